"""Run one GEMM shape (for ncu): M N K a_kmajor b_kmajor epi c_bf16 [iters]."""
import ctypes as C
import sys

sys.path.insert(0, "/root/repo")
import torch  # noqa: E402

from paper_2411_02908_b200 import _capi as A  # noqa: E402

m, n, k, ak, bk, epi, cb = (int(x) for x in sys.argv[1:8])
iters = int(sys.argv[8]) if len(sys.argv) > 8 else 2
a = torch.randn(m * k, device="cuda").bfloat16()
b = torch.randn(k * n, device="cuda").bfloat16()
c = torch.zeros(m * n, device="cuda", dtype=torch.bfloat16 if cb else torch.float32)
bias = torch.zeros(n, device="cuda")
resid = torch.zeros(m * n, device="cuda") if epi == 3 else None
aux = torch.zeros(m * n, device="cuda").bfloat16() if epi in (4, 5) else None
ms = C.c_double()
err = A.photon_err()
rc = A.lib().photon_debug_gemm(1, m, n, k, a.data_ptr(), k if ak else m, ak, b.data_ptr(),
                               k if bk else n, bk, 1, c.data_ptr(), n, cb, epi, bias.data_ptr(),
                               resid.data_ptr() if resid is not None else None,
                               aux.data_ptr() if aux is not None else None, iters, C.byref(ms),
                               C.byref(err))
assert rc == 0, err.msg
print(f"{ms.value*1e3:.1f} us  {2.0*m*n*k/ms.value/1e9:.1f} TF/s")
