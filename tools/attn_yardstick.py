"""Attention yardstick at the 125M shape (B=32, H=12, S=2048, dh=64, causal,
bf16): our tcgen05 kernels (photon_debug_attention impl 2) next to torch SDPA's
cuDNN and flash backends on the same box.  A calibration only: library
attention is never on the product path.  FLOPs: forward 4*B*H*dh*S(S+1)/2,
backward counted as 2.5x forward.

    python tools/attn_yardstick.py [--dh 64|128]
"""
import argparse
import ctypes as C
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402
import torch.nn.functional as Fn  # noqa: E402
from torch.nn.attention import SDPBackend, sdpa_kernel  # noqa: E402

from paper_2411_02908_b200 import _capi as A  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--dh", type=int, default=64)
args = ap.parse_args()
dh = args.dh
B, S, H = (32, 2048, 12) if dh == 64 else (16, 2048, 16)
d = H * dh
flops = 4.0 * B * H * dh * S * (S + 1) / 2


def ev_time(fn, reps=5):
    fn()
    torch.cuda.synchronize()
    ts = []
    for _ in range(reps):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        fn()
        e1.record()
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1))
    ts.sort()
    return ts[len(ts) // 2]


# ours: [B*S, d] row-major, head h in columns [h*dh, (h+1)*dh)
q, k, v, dO = (torch.randn(B * S, d, device="cuda").bfloat16() for _ in range(4))
o = torch.empty_like(q)
dq, dk, dv = torch.empty_like(q), torch.empty_like(q), torch.empty_like(q)
lse = torch.empty(B * H * S, device="cuda")
scr = torch.empty(B * H * S, device="cuda")
err = A.photon_err()
lib = A.lib()


def ours(bwd):
    ms = C.c_double()
    rc = lib.photon_debug_attention(2, B, S, H, d, q.data_ptr(), k.data_ptr(), v.data_ptr(),
                                    o.data_ptr(), lse.data_ptr(),
                                    dO.data_ptr() if bwd else None, scr.data_ptr() if bwd else None,
                                    dq.data_ptr() if bwd else None, dk.data_ptr() if bwd else None,
                                    dv.data_ptr() if bwd else None, C.byref(ms), C.byref(err))
    assert rc == 0, err.msg
    return ms.value


ours(False)
f_ours = sorted(ours(False) for _ in range(5))[2]
ours(True)
b_ours = sorted(ours(True) for _ in range(5))[2]
print(f"ours (tcgen05)   fwd {f_ours:.3f} ms {flops / f_ours / 1e9:6.1f} TF/s   "
      f"bwd {b_ours:.3f} ms {2.5 * flops / b_ours / 1e9:6.1f} TF/s", flush=True)

# torch SDPA: [B, H, S, dh]
qt = q.view(B, S, H, dh).transpose(1, 2).contiguous().requires_grad_(True)
kt = k.view(B, S, H, dh).transpose(1, 2).contiguous().requires_grad_(True)
vt = v.view(B, S, H, dh).transpose(1, 2).contiguous().requires_grad_(True)
gt = dO.view(B, S, H, dh).transpose(1, 2).contiguous()
for name, be in (("cudnn", SDPBackend.CUDNN_ATTENTION), ("flash", SDPBackend.FLASH_ATTENTION)):
    try:
        with sdpa_kernel([be]):
            out = Fn.scaled_dot_product_attention(qt, kt, vt, is_causal=True)
            f = ev_time(lambda: Fn.scaled_dot_product_attention(qt, kt, vt, is_causal=True))

            def fb():
                y = Fn.scaled_dot_product_attention(qt, kt, vt, is_causal=True)
                y.backward(gt)

            fbt = ev_time(fb)
        bt = fbt - f
        print(f"sdpa {name:7s}     fwd {f:.3f} ms {flops / f / 1e9:6.1f} TF/s   "
              f"bwd {bt:.3f} ms {2.5 * flops / bt / 1e9:6.1f} TF/s  (fwd+bwd {fbt:.3f})",
              flush=True)
    except Exception as ex:  # backend unavailable on this build
        print(f"sdpa {name}: unavailable ({str(ex)[:120]})", flush=True)
