"""Weight-gradient GEMM time by operand layout (photon_debug_gemm, tcgen05, fp32
out): dW = X^T G over K = 65,536 tokens with X / G either MN-major (the
activations as stored) or K-major (a transposed copy)."""
import ctypes as C
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2411_02908_b200 import _capi as A  # noqa: E402

lib, err = A.lib(), A.photon_err()
K = 65536
for M, N in ((768, 768), (768, 3072), (3072, 768)):
    x = torch.randn(K, M, device="cuda").bfloat16()   # activations [tokens, M]
    g = torch.randn(K, N, device="cuda").bfloat16()   # gradients [tokens, N]
    xt, gt = x.t().contiguous(), g.t().contiguous()
    c = torch.empty(M, N, device="cuda")
    for ak, bk in ((False, False), (True, False), (False, True), (True, True)):
        Ap, lda = (xt, K) if ak else (x, M)
        Bp, ldb = (gt, K) if bk else (g, N)
        ms = C.c_double()
        rc = lib.photon_debug_gemm(1, M, N, K, Ap.data_ptr(), lda, int(ak), Bp.data_ptr(), ldb, int(bk),
                                   1, c.data_ptr(), N, 0, 0, None, None, None, 10, C.byref(ms),
                                   C.byref(err))
        assert rc == 0, err.msg
        print(f"{M}x{N}x{K}  A {'K' if ak else 'MN'}-major  B {'K' if bk else 'MN'}-major: "
              f"{ms.value * 1e3:.1f} us  {2 * M * N * K / ms.value / 1e9:.0f} TF/s", flush=True)
