"""Time tcgen05 attention fwd/bwd at the Photon-1.3B head shape (dh = 128, S = 2048)."""
import ctypes as C
import sys

sys.path.insert(0, "/root/repo")
import torch  # noqa: E402

from paper_2411_02908_b200 import _capi as A  # noqa: E402

B, S, H = int(sys.argv[1]) if len(sys.argv) > 1 else 16, 2048, 16
d = 128 * H
q, k, v, dO = (torch.randn(B * S * d, device="cuda").bfloat16() for _ in range(4))
o = torch.empty_like(q)
dq, dk, dv = torch.empty_like(q), torch.empty_like(q), torch.empty_like(q)
lse = torch.empty(B * H * S, device="cuda")
scr = torch.empty(B * H * S, device="cuda")
err = A.photon_err()
flops = 4.0 * B * H * 128 * S * (S + 1) / 2
for impl in (1, 2):
    ms = C.c_double()
    for _ in range(3):
        A.lib().photon_debug_attention(impl, B, S, H, d, q.data_ptr(), k.data_ptr(), v.data_ptr(),
                                       o.data_ptr(), lse.data_ptr(), None, None, None, None, None,
                                       C.byref(ms), C.byref(err))
    print(f"fwd impl {impl}: {ms.value:.3f} ms  {flops/ms.value/1e9:.1f} TF/s", flush=True)
    for _ in range(3):
        A.lib().photon_debug_attention(impl, B, S, H, d, q.data_ptr(), k.data_ptr(), v.data_ptr(),
                                       o.data_ptr(), lse.data_ptr(), dO.data_ptr(), scr.data_ptr(),
                                       dq.data_ptr(), dk.data_ptr(), dv.data_ptr(), C.byref(ms),
                                       C.byref(err))
    print(f"bwd impl {impl}: {ms.value:.3f} ms  {2.5*flops/ms.value/1e9:.1f} TF/s (2.5x fwd flops)",
          flush=True)
