"""Our tcgen05 attention at the 125M shape (B=32 H=12 S=2048 dh=64, causal):
forward and backward device time, median of 7 (use PHOTON_LIB for variants)."""
import ctypes as C
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2411_02908_b200 import _capi as A  # noqa: E402

dh = int(os.environ.get("ATTN_DH", "64"))
B, S, H = (32, 2048, 12) if dh == 64 else (16, 2048, 16)
d = H * dh
q, k, v, dO = (torch.randn(B * S, d, device="cuda").bfloat16() for _ in range(4))
o = torch.empty_like(q)
dq, dk, dv = torch.empty_like(q), torch.empty_like(q), torch.empty_like(q)
lse = torch.empty(B * H * S, device="cuda")
err = A.photon_err()
lib = A.lib()


def run(bwd):
    ms = C.c_double()
    rc = lib.photon_debug_attention(2, B, S, H, d, q.data_ptr(), k.data_ptr(), v.data_ptr(),
                                    o.data_ptr(), lse.data_ptr(), dO.data_ptr() if bwd else None,
                                    None, dq.data_ptr() if bwd else None,
                                    dk.data_ptr() if bwd else None, dv.data_ptr() if bwd else None,
                                    C.byref(ms), C.byref(err))
    assert rc == 0, err.msg
    return ms.value


f = sorted(run(False) for _ in range(7))[3]
b = sorted(run(True) for _ in range(7))[3]
fl = 4.0 * B * H * dh * S * (S + 1) / 2
print(f"{os.path.basename(A.LIB_PATH)} dh={dh}: fwd {f:.3f} ms {fl / f / 1e9:.0f} TF/s  "
      f"bwd {b:.3f} ms {2.5 * fl / b / 1e9:.0f} TF/s", flush=True)
