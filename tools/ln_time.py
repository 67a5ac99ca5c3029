"""LayerNorm forward (and forward+backward) device time at the 125M shape
(M = 65,536, d = 768, bf16 output), median of 9; PHOTON_LIB selects a variant."""
import ctypes as C
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2411_02908_b200 import _capi as A  # noqa: E402

M, d = 65536, int(os.environ.get("LN_D", "768"))
x, dres = (torch.randn(M, d, device="cuda") for _ in range(2))
dy = torch.randn(M, d, device="cuda").bfloat16()  # the dX GEMMs write bf16
g, b = torch.randn(d, device="cuda"), torch.randn(d, device="cuda")
y = torch.empty(M, d, device="cuda", dtype=torch.bfloat16)
mean, rstd = torch.empty(M, device="cuda"), torch.empty(M, device="cuda")
dx = torch.empty(M, d, device="cuda")
dxT = torch.empty(M, d, device="cuda", dtype=torch.bfloat16)
dg, db, ds = (torch.empty(d, device="cuda") for _ in range(3))
lib, err = A.lib(), A.photon_err()
P = lambda t: t.data_ptr()  # noqa: E731


def run(bwd):
    ms = C.c_double()
    rc = lib.photon_debug_layernorm(1, M, d, P(x), P(g), P(b), P(y), P(mean), P(rstd),
                                    P(dy) if bwd else None, P(dres), P(dx), P(dxT), P(dg), P(db),
                                    P(ds), C.byref(ms), C.byref(err))
    assert rc == 0, err.msg
    return ms.value


f = sorted(run(False) for _ in range(9))[4]
fb = sorted(run(True) for _ in range(9))[4]
print(f"{os.path.basename(A.LIB_PATH)} d={d}: fwd {f * 1e3:.1f} us ({M * d * 6 / f / 1e6:.0f} GB/s)  "
      f"fwd+bwd {fb * 1e3:.1f} us", flush=True)
