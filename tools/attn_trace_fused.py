"""Timeline of the fused HD = 64 backward (CTA 0, its first 64 tiles) from the
instrumented build (events 20-29).
  PHOTON_BUILD_TRACE=1 python -m paper_2411_02908_b200.build
  PHOTON_LIB=paper_2411_02908_b200/libphoton_trace.so python tools/attn_trace_fused.py"""
import ctypes as C
import sys

sys.path.insert(0, "/root/repo")
import torch  # noqa: E402

from paper_2411_02908_b200 import _capi as A  # noqa: E402

B, S, H, d = 32, 2048, 12, 768
q, k, v, dO = (torch.randn(B * S * d, device="cuda").bfloat16() for _ in range(4))
o = torch.empty_like(q)
dq, dk, dv = torch.empty_like(q), torch.empty_like(q), torch.empty_like(q)
lse = torch.empty(B * H * S, device="cuda")
err = A.photon_err()
ms = C.c_double()
for bwd in (False, True, True):
    A.lib().photon_debug_attention(2, B, S, H, d, q.data_ptr(), k.data_ptr(), v.data_ptr(),
                                   o.data_ptr(), lse.data_ptr(), dO.data_ptr() if bwd else None,
                                   None, dq.data_ptr() if bwd else None,
                                   dk.data_ptr() if bwd else None, dv.data_ptr() if bwd else None,
                                   C.byref(ms), C.byref(err))
torch.cuda.synchronize()
print(f"backward {ms.value:.3f} ms")
buf = (C.c_ulonglong * (64 * 64))()
assert A.lib().photon_debug_attn_trace(buf, 64 * 64) == 0
names = "prod_q,mma_qfull,mma_sissue,mma_grads,sm_lastload,sm_sfull,sm_computed,sm_pvdone,sm_pfull,sm_emitted,max_comp,max_emit".split(",")
base = 20
t0 = min(buf[(base + e) * 64] for e in range(len(names)) if buf[(base + e) * 64])
print("g  " + " ".join(f"{n:>11s}" for n in names))
prev = None
for g in range(64):
    row = [buf[(base + e) * 64 + g] for e in range(len(names))]
    print(f"{g:2d} " + " ".join(f"{(x - t0) if x else -1:11d}" for x in row))
