"""Time the cross-entropy pass at the 125M head shape (M = 65,536, V = 50,368):
with the head-bias column sums accumulated inside it (tensor memory) vs the
pass without them followed by the separate column-sum kernel (photon_debug_ce /
photon_debug_colsum, device time per call, median of 5)."""
import ctypes as C
import os
import statistics
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2411_02908_b200 import _capi as A  # noqa: E402

M, V = int(os.environ.get("CE_M", 65536)), 50368
lib = A.lib()
g = torch.Generator(device="cuda").manual_seed(0)
base = (torch.randn(M, V, device="cuda", generator=g) * 2).bfloat16()
tgt = torch.randint(0, V, (M,), device="cuda", generator=g, dtype=torch.int32)
buf = torch.empty_like(base)
rowloss = torch.zeros(M, device="cuda", dtype=torch.float64)
dbias = torch.zeros(V, device="cuda")
ms, err = C.c_double(), A.photon_err()


def run(fused):
    t = []
    for _ in range(6):
        buf.copy_(base)
        torch.cuda.synchronize()
        rc = lib.photon_debug_ce(buf.data_ptr(), 1, tgt.data_ptr(), M, V, C.c_float(1.0 / M),
                                 rowloss.data_ptr(), 1, dbias.data_ptr() if fused else None,
                                 C.byref(ms), C.byref(err))
        assert rc == 0, err.msg
        tot = ms.value
        if not fused:
            rc = lib.photon_debug_colsum(buf.data_ptr(), 1, M, V, dbias.data_ptr(), C.byref(ms),
                                         C.byref(err))
            assert rc == 0, err.msg
            tot += ms.value
        t.append(tot)
    return statistics.median(t[1:])


a = run(False)
b = run(True)
gb = 2 * M * V * 2 / 1e9
print(f"CE + column-sum pass: {a:.3f} ms   CE with fused bias sums: {b:.3f} ms   "
      f"(CE algorithmic {gb:.1f} GB -> {gb / b:.2f} TB/s fused)")
