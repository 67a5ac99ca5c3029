"""aggregation-only sweep at N in {164.04M, 1,419.15M,
6,865.22M} parameters (fp32), outer Nesterov (eta 0.1, mu 0.9).

  python tools/agg_sweep.py                  # 1 GPU: all K client models in HBM
  torchrun --nproc-per-node G tools/agg_sweep.py   # G GPUs: 1 client per GPU,
        # the runner's sharded boundary (NCCL exchange -> fused update -> all-gather)

One JSON line per N (rank 0).  Single GPU: algorithmic HBM bytes (K+4)*N*4 /
time vs the measured HBM copy bandwidth.  G GPUs: per-GPU wire bytes
2(G-1)/G*N*4 / time ("busbw") vs 900 GB/s NVLink 5, time = max over ranks."""
import ctypes as C
import json
import os
import statistics
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
os.environ.setdefault("NCCL_DEBUG", "WARN")
import torch  # noqa: E402

from paper_2411_02908_b200 import _capi as A  # noqa: E402
from paper_2411_02908_b200 import fedsim as F  # noqa: E402

NS = [int(x) for x in os.environ.get("PHOTON_AGG_NS", "164044480,1419154624,6865216704").split(",")]
world = int(os.environ.get("WORLD_SIZE", "1"))
rank = int(os.environ.get("RANK", "0"))
local = int(os.environ.get("LOCAL_RANK", "0"))
torch.cuda.set_device(local)
srv = F.ServerOptConfig(1, 0.1, 0.9, True).c()
peaks = {}
try:
    peaks = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))
except Exception:
    pass
hbm = float(peaks.get("hbm_copy_gbs", peaks.get("hbm_gbs", 6555.2)) or 6555.2) \
    if isinstance(peaks, dict) else 6555.2

if world == 1:
    ctx = F.context(F.ModelConfig(1, 32, 2, 4, 64, 16), local, "f32", 1)
    for n in NS:
        k = max(1, min(8, int(150e9 / (4 * n)) - 2))
        dev = torch.device("cuda", local)
        models = [torch.zeros(n, device=dev) for _ in range(k)]
        theta = torch.zeros(n, device=dev)
        vel = torch.zeros(n, device=dev)
        ptrs = (C.c_void_p * k)(*[m.data_ptr() for m in models])
        ms = C.c_double()
        times = []
        for i in range(7):
            F._call(A.lib().photon_aggregate_device_f32, ctx.handle, ptrs, k, n,
                    C.c_void_p(theta.data_ptr()), C.c_void_p(vel.data_ptr()), C.byref(srv),
                    C.byref(ms))
            if i >= 2:
                times.append(ms.value)
        t = statistics.median(times)
        nbytes = (k + 4) * n * 4
        print(json.dumps({"variant": "single-gpu HBM", "n_params": n, "clients": k, "ms": t,
                          "algorithmic_bytes": nbytes, "achieved_gbs": nbytes / t / 1e6,
                          "peak_gbs": hbm, "frac": nbytes / t / 1e6 / hbm}), flush=True)
        del models, theta, vel
        torch.cuda.empty_cache()
else:
    import torch.distributed as dist

    dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    for n in NS:
        obj = [F.nccl_unique_id() if rank == 0 else None]  # a fresh id per communicator
        dist.broadcast_object_list(obj, src=0)
        idbuf = (C.c_uint8 * 128).from_buffer_copy(obj[0])
        ms = C.c_double()
        F._call(A.lib().photon_debug_boundary, local, n, rank, world, idbuf, C.byref(srv), 5,
                C.byref(ms))
        t = torch.tensor([ms.value], device="cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        tmax = float(t.item())
        wire = 2 * (world - 1) / world * n * 4
        if rank == 0:
            print(json.dumps({"variant": f"sharded boundary on {world} GPUs (1 client/GPU)",
                              "n_params": n, "ms_max_over_ranks": tmax,
                              "wire_bytes_per_gpu": wire, "busbw_gbs": wire / tmax / 1e6,
                              "nvlink_gbs": 900.0, "frac": wire / tmax / 1e6 / 900.0,
                              "owner_hbm_bytes": (world + 4) * n / world * 4}), flush=True)
    dist.barrier()
    dist.destroy_process_group()
