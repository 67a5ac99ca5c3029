"""Time the client-step contractions at the 125M shape through photon_debug_gemm."""
import ctypes as C
import sys

sys.path.insert(0, "/root/repo")
import torch  # noqa: E402

from paper_2411_02908_b200 import _capi as A  # noqa: E402

M, d, hid, V = 65536, 768, 3072, 50368
# name, M, N, K, a_kmajor, b_kmajor, epi, c_bf16
CASES = [
    ("fwd qkv  [M,d]x[d,d] +b", M, d, d, 1, 0, 2, 1),
    ("fwd o    +b +resid f32", M, d, d, 1, 0, 3, 0),
    ("fwd w1   +b gelu", M, hid, d, 1, 0, 4, 1),
    ("fwd w1   +b (no gelu)", M, hid, d, 1, 0, 2, 1),
    ("fwd w1   store", M, hid, d, 1, 0, 0, 1),
    ("fwd w2   +b +resid", M, d, hid, 1, 0, 3, 0),
    ("fwd head +b", M, V, d, 1, 0, 2, 1),
    ("dX  w2   gelu'", M, hid, d, 1, 1, 5, 1),
    ("dX  w1   f32", M, d, hid, 1, 1, 0, 0),
    ("dX  head f32", M, d, V, 1, 1, 0, 0),
    ("dX  dxd  accum f32", M, d, d, 1, 1, 1, 0),
    ("dW  dxd  (split-K)", d, d, M, 0, 0, 0, 0),
    ("dW  w2", hid, d, M, 0, 0, 0, 0),
    ("dW  w1", d, hid, M, 0, 0, 0, 0),
    ("dW  head", d, V, M, 0, 0, 0, 0),
    # layout / fusion probes: the dW shapes with K-major operands, one N = 3d qkv
    ("probe dW dxd K-major", d, d, M, 1, 1, 0, 0),
    ("probe dW w1 K-major", d, hid, M, 1, 1, 0, 0),
    ("probe fwd qkv N=3d +b", M, 3 * d, d, 1, 0, 2, 1),
    ("probe dW head A K-major", d, V, M, 1, 0, 0, 0),
    ("probe fwd head B K-major +b", M, V, d, 1, 1, 2, 1),
    ("probe fwd w1 B K-major +b gelu", M, hid, d, 1, 1, 4, 1),
    ("probe fwd qkv B K-major +b", M, d, d, 1, 1, 2, 1),
    ("probe fwd w2 B K-major +b +resid", M, d, hid, 1, 1, 3, 0),
    ("probe dW w1 A K-major", d, hid, M, 1, 0, 0, 0),
    ("probe dW w2 A K-major", hid, d, M, 1, 0, 0, 0),
]
if len(sys.argv) > 2:  # only the cases whose name contains argv[2]
    CASES = [c for c in CASES if sys.argv[2] in c[0]]
impl = int(sys.argv[1]) if len(sys.argv) > 1 else 1
tot_f, tot_t = 0.0, 0.0
for name, m, n, k, ak, bk, epi, cb in CASES:
    a = torch.randn(m * k, device="cuda").bfloat16()
    b = torch.randn(k * n, device="cuda").bfloat16()
    c = torch.zeros(m * n, device="cuda", dtype=torch.bfloat16 if cb else torch.float32)
    bias = torch.zeros(n, device="cuda")
    resid = torch.zeros(m * n, device="cuda") if epi == 3 else None
    aux = torch.zeros(m * n, device="cuda").bfloat16() if epi in (4, 5) else None
    lda = k if ak else m
    ldb = k if bk else n
    ms = C.c_double()
    err = A.photon_err()
    args = (impl, m, n, k, a.data_ptr(), lda, ak, b.data_ptr(), ldb, bk, 1, c.data_ptr(), n, cb, epi,
            bias.data_ptr(), resid.data_ptr() if resid is not None else None,
            aux.data_ptr() if aux is not None else None)
    A.lib().photon_debug_gemm(*args, 3, C.byref(ms), C.byref(err))
    rc = A.lib().photon_debug_gemm(*args, 10, C.byref(ms), C.byref(err))
    assert rc == 0, err.msg
    fl = 2.0 * m * n * k
    tot_f += fl
    tot_t += ms.value
    print(f"{name:28s} M={m:6d} N={n:6d} K={k:6d}  {ms.value*1e3:8.1f} us  {fl/ms.value/1e9:7.1f} TF/s",
          flush=True)
print(f"aggregate {tot_f/tot_t/1e9:.1f} TF/s")
