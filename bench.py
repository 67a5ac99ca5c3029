#!/usr/bin/env python
"""Benchmark: one Photon federated round per step (BASELINE.json configs[1]).

Workload: the reference architecture at the Photon-125M shape (L12 d768 H12 e4
V50368 S2048, 164.04 M params), one client per GPU (weak scaling: K = N
clients), B = 32, tau local AdamW steps, then the anchored FedAvg + outer
Nesterov step (eta 0.1, mu 0.9) at the round boundary.  A step = one round;
tokens/round = K * tau * B * S.

  value  tokens/s of the whole job, device-timed (CUDA events from the first
         local step to theta_{t+1} on every GPU; inputs resident in HBM), max
         over ranks.
  e2e    the same metric through the public API (FederationRunner.run_round):
         host BatchStream staging, pinned H2D of the round's tokens, the round,
         D2H of the step losses -- wall clock, max over ranks.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--tau T] [--impl reference]
"""
from __future__ import annotations

import argparse
import ctypes as C
import json
import os
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)
# stdout carries exactly one JSON line: the line goes to a private copy of the
# original stdout, and fd 1 is pointed at stderr so that banners printed by
# native libraries (NCCL's version line, ...) cannot reach the driver's parser
_JSON_OUT = os.fdopen(os.dup(1), "w")
os.dup2(2, 1)


def _emit(line: dict) -> None:
    _JSON_OUT.write(json.dumps(line) + "\n")
    _JSON_OUT.flush()

MODEL_125M = (12, 768, 12, 4, 50368, 2048)
# SURVEY 8(d) configs 2-4 (Photon 125M / 1.3B / 7B, reference architecture)
MODELS = {"125m": (MODEL_125M, "Photon-125M", "164.04M"),
          "1.3b": ((24, 2048, 16, 4, 50368, 2048), "Photon-1.3B", "1,419.15M"),
          "7b": ((32, 4096, 32, 4, 50368, 2048), "Photon-7B", "6,865.22M")}
MEASURED_PEAKS = os.path.join(ROOT, "MEASURED_PEAKS.json")
METRIC = "tokens/s/round at 1-8 B200 (125M); FedAvg aggregate GB/s vs roofline"


NCU_GEMM = os.path.join(ROOT, "profiles", "r01_ncu_gemm_dram.json")


def _gemm_traffic():
    """Mean DRAM bytes (read + write) per gemm_tc launch over the GEMM launches
    of one 125M client step, from the committed ncu capture
    (tools/capture_profiles.sh -> profiles/r01_ncu_gemm_dram.json), or None."""
    try:
        with open(NCU_GEMM) as f:
            ks = json.load(f)["kernels"]
        n = sum(v["launches"] for k, v in ks.items() if "gemm_tc" in k)
        b = sum(v["launches"] * v["dram_bytes_per_launch"] for k, v in ks.items() if "gemm_tc" in k)
        return b / n if n else None
    except Exception:
        return None


def _boundary_path(n_params: int) -> str:
    """Which boundary the runner takes (runner.cpp use_peer_boundary): NVLink peer
    memory up to 24 GB per fp32 replica, NCCL beyond or when forced."""
    forced = os.environ.get("PHOTON_BOUNDARY")
    if forced in ("nccl", "p2p"):
        return forced
    return "p2p" if n_params * 4 <= 24e9 else "nccl"


def _peaks():
    try:
        with open(MEASURED_PEAKS) as f:
            p = json.load(f)
        return p["hbm_gbs"], p["bf16_tflops"], p["bf16_tflops_sustained"], "measured"
    except Exception:
        return 6650.0, 1590.0, 1400.0, "fallback"


# ---------------------------------------------------------------------------
# clocks during the timed region
# ---------------------------------------------------------------------------
class ClockSampler:
    FIELDS = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, device: int):
        self.device = device
        self.rows = []
        self._proc = None

    def __enter__(self):
        try:
            self._proc = subprocess.Popen(
                ["nvidia-smi", f"--id={self.device}", f"--query-gpu={self.FIELDS}",
                 "--format=csv,noheader,nounits", "-lms", "200"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self._t = threading.Thread(target=self._read, daemon=True)
            self._t.start()
        except Exception:
            self._proc = None
        return self

    def _read(self):
        for line in self._proc.stdout:
            parts = [p.strip() for p in line.split(",")]
            if len(parts) >= 9:
                self.rows.append(parts)

    def __exit__(self, *exc):
        if self._proc:
            self._proc.terminate()
            try:
                self._proc.wait(timeout=5)
            except Exception:
                self._proc.kill()

    def summary(self):
        if not self.rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"]}
        sm = [float(r[1]) for r in self.rows if r[1].replace(".", "").isdigit()]
        mx = [float(r[2]) for r in self.rows if r[2].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({n for r in self.rows for n, v in zip(names, r[5:9]) if v == "Active"})
        loaded = [s for s in sm if s > 0.5 * (max(mx) if mx else 1)] or sm
        return {"sm_mhz": statistics.median(loaded) if loaded else None,
                "sm_max_mhz": max(mx) if mx else None, "reasons": reasons,
                "samples": len(self.rows)}


# ---------------------------------------------------------------------------
# distributed plumbing (torch.distributed over NCCL: barrier, max, id exchange)
# ---------------------------------------------------------------------------
def _dist_setup(n_gpus: int):
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world > 1:
        import torch
        import torch.distributed as dist

        torch.cuda.set_device(local)
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    return rank, world, local


def _barrier(world):
    if world > 1:
        import torch.distributed as dist

        dist.barrier()


def _max_over_ranks(vals, world, local):
    if world == 1:
        return list(vals)
    import torch
    import torch.distributed as dist

    t = torch.tensor(list(vals), dtype=torch.float64, device=f"cuda:{local}")
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return t.tolist()


def _bcast_bytes(b: bytes, world, local):
    if world == 1:
        return b
    import torch.distributed as dist

    obj = [b]
    dist.broadcast_object_list(obj, src=0)
    return obj[0]


# ---------------------------------------------------------------------------
# CPU baseline: the reference's own client step (oracle/_ref) on host cores
# ---------------------------------------------------------------------------
def _cpu_threads():
    n = os.cpu_count() or 1
    try:
        with open("/proc/meminfo") as f:
            avail_kb = next(int(l.split()[1]) for l in f if l.startswith("MemAvailable"))
        by_mem = max(1, int(avail_kb / 1024 / 1024 / 9))  # ~7-8 GB per 125M f64 client
    except Exception:
        by_mem = 4
    return max(1, min(n, by_mem, 64))


def cpu_sample(seq: int = 32, threads: int | None = None):
    """(tokens/s, cores, kind, sample description) of the reference CPU path."""
    from oracle import ModelCfg, TrainCfg, load_reference

    threads = threads or _cpu_threads()
    ref = load_reference()
    mc = ModelCfg(*MODEL_125M)
    t = TrainCfg(eta_max=6e-4, warmup_steps=64, decay_steps=1024, alpha=0.1, batch_size=1)
    if ref is not None:
        secs, _ = ref.train_sample(mc, t, 1, seq, 1, threads)
        kind = "reference"
    else:  # the C restatement, single thread per client (oracle port)
        import numpy as np

        from oracle import load_oracle

        o = load_oracle()
        p = o.init_params(mc, 1)
        corpus = o.generate_corpus("web", 4 * (seq + 1), 7, mc.vocab_size)
        t0 = time.perf_counter()
        o.forward_backward(mc, p, corpus[:seq].astype(np.int32), corpus[1:seq + 1].astype(np.int32),
                           1, seq)
        secs = time.perf_counter() - t0
        threads = 1
        kind = "port"
    tokens = threads * seq
    sample = (f"{threads} reference clients x 1 local AdamW step, B=1 x S={seq} tokens each, "
              f"125M reference architecture (f64, {threads} host threads)")
    return tokens / secs, threads, kind, sample


def run_reference_arm(args):
    rank, world, local = _dist_setup(args.gpus)
    if rank != 0:
        return 0
    # bounded samples of the reference's own CPU client step; one per "step"
    for _ in range(args.warmup):
        cpu_sample(args.cpu_seq)
    vals = []
    t0 = time.perf_counter()
    for _ in range(args.steps):
        v, cores, kind, sample = cpu_sample(args.cpu_seq)
        vals.append(v)
    wall = time.perf_counter() - t0
    value = statistics.median(vals)
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": "tokens/s",
        "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": 1000.0 * wall / max(args.steps, 1), "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": dict(_config(args), precision="f64 (the reference's own arithmetic)"),
        "cpu_baseline": {"value": value, "unit": "tokens/s", "cores": cores, "kind": kind,
                         "sample": sample},
        "e2e": {"value": value, "unit": "tokens/s", "h2d_bytes_per_step": 0,
                "d2h_bytes_per_step": 0},
    }
    _emit(line)
    return 0


def _config(args):
    shape, name, params = MODELS[args.model]
    L, d, H, e, V, S = shape
    return {"workload": f"{name} federated round (reference architecture, {params} params)",
            "model": f"L{L} d{d} H{H} e{e} V{V} S{S}", "clients": args.gpus,
            "clients_per_gpu": 1, "local_steps": args.tau, "batch": args.batch, "seq_len": S,
            "global_batch": args.gpus * args.batch, "server_opt": "nesterov eta=0.1 mu=0.9",
            "parallelism": f"fed{args.gpus}", "precision": args.precision,
            "l2": "inputs larger than L2 (weights+activations >> 126 MB)"}


# ---------------------------------------------------------------------------
# aggregation-only sweep (BASELINE config 5, single GPU)
# ---------------------------------------------------------------------------
def aggregation_sweep(ctx, n_params: int, k: int, iters: int = 5):
    import torch

    from paper_2411_02908_b200 import _capi as A
    from paper_2411_02908_b200.fedsim import ServerOptConfig, _call

    dev = torch.device("cuda", ctx.device)
    models = [torch.randn(n_params, device=dev) * 0.02 for _ in range(k)]
    theta = torch.randn(n_params, device=dev) * 0.02
    vel = torch.zeros(n_params, device=dev)
    ptrs = (C.c_void_p * k)(*[m.data_ptr() for m in models])
    cfg = ServerOptConfig(1, 0.1, 0.9, True).c()
    ms = C.c_double()
    times = []
    for i in range(iters + 2):
        _call(A.lib().photon_aggregate_device_f32, ctx.handle, ptrs, k, n_params,
              C.c_void_p(theta.data_ptr()), C.c_void_p(vel.data_ptr()), C.byref(cfg),
              C.byref(ms))
        if i >= 2:
            times.append(ms.value)
    t = statistics.median(times)
    nbytes = (k + 4) * n_params * 4  # read k models + theta + v, write theta + v
    return nbytes / (t * 1e-3) / 1e9, t, nbytes


# ---------------------------------------------------------------------------
# our arm
# ---------------------------------------------------------------------------
def run_ours(args):
    rank, world, local = _dist_setup(args.gpus)
    import numpy as np

    from paper_2411_02908_b200 import _capi as A
    from paper_2411_02908_b200 import fedsim as F

    hbm, bf16_burst, bf16_sus, peak_src = _peaks()
    L, d, H, e, V, S = MODELS[args.model][0]
    model = F.ModelConfig(L, d, H, e, V, S)
    K = world  # weak scaling: one client per GPU
    rounds = args.warmup + args.steps + 1
    tau, B = args.tau, args.batch
    # corpus: one epoch per client per round of tau*B blocks of S+1 tokens
    n_tok = K * tau * B * (S + 1) + S + 1
    corpus = F.generate_corpus("web", n_tok, 7, V)
    plan = F.partition_iid(corpus, K, S, 7)
    theta0 = F.TransformerModel(model).init_params(1)
    local_cfg = F.LocalTrainConfig(model=model, schedule=F.LrSchedule(6e-4, 64, 1024, 0.1),
                                   local_steps=tau, batch_size=B)
    server = F.ServerOptConfig(1, 0.1, 0.9, True)
    nccl_id = _bcast_bytes(F.nccl_unique_id() if rank == 0 else b"", world, local) \
        if world > 1 else None
    runner = F.FederationRunner(F.FederationConfig(K, K, rounds, F.Topology.kRingAllReduce, 42),
                                local_cfg, server, plan, theta0, device=local,
                                precision=args.precision, rank=rank, world=world,
                                nccl_id=nccl_id)
    for _ in range(args.warmup):
        runner.run_round()

    # ---- timed region: K rounds, barrier + sync on both sides
    import torch

    torch.cuda.synchronize(local)
    _barrier(world)
    dev_ms, recs = 0.0, []
    with ClockSampler(local) as clk:
        t0 = time.perf_counter()
        for _ in range(args.steps):
            rec = runner.run_round()
            recs.append(rec)
            dev_ms += rec.round_ms
        torch.cuda.synchronize(local)
        wall = time.perf_counter() - t0
    _barrier(world)
    agg_ms = sum(r.boundary_ms for r in recs) / max(len(recs), 1)
    dev_ms_max, wall_max, agg_ms_max = _max_over_ranks([dev_ms, wall, agg_ms], world, local)
    tokens_total = K * tau * B * S * args.steps
    value = tokens_total / (dev_ms_max / 1000.0)
    e2e = tokens_total / wall_max

    # ---- kernel-class timing in one instrumented round (not part of value)
    prof = {}
    lib = A.lib()
    if hasattr(lib, "photon_ctx_set_timing"):
        times = (C.c_double * 8)()
        lib.photon_ctx_set_timing(runner.ctx.handle, 1)
        runner.run_round()
        lib.photon_ctx_kernel_times(runner.ctx.handle, times)
        lib.photon_ctx_set_timing(runner.ctx.handle, 0)
        prof = {"gemm_ms": times[0], "attn_ms": times[1], "other_ms": times[2],
                "gemm_flops": times[3], "attn_flops": times[4], "gemm_launches": times[5],
                "attn_launches": times[6], "launches": times[7]}

    agg = None
    if rank == 0 and not args.no_agg:
        import torch

        P = model.param_count()
        # the side measurement needs (k + 2) * P fp32 beside the resident engine;
        # at 7B that leaves room for few (or no) client models -- shrink k, never OOM
        free, _ = torch.cuda.mem_get_info(runner.ctx.device)
        k_fit = min(args.agg_k, int((free - (2 << 30)) // (4 * P)) - 2)
        if k_fit >= 2:
            gbs, ms, nbytes = aggregation_sweep(runner.ctx, P, k_fit)
            agg = {"n_params": P, "clients": k_fit,
                   "kernel": "fused anchored-mean+nesterov f32", "ms": ms,
                   "algorithmic_bytes": nbytes, "achieved_gbs": gbs, "peak_gbs": hbm,
                   "frac": gbs / hbm}

    if rank != 0:
        return 0
    flops_per_token = 3 * (2 * (L * (4 + 2 * e) * d * d + d * V) + 4 * L * d * (S + 1) / 2)
    rec0 = recs[-1]
    line = {
        "metric": METRIC, "value": value, "unit": "tokens/s", "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": dev_ms_max / max(args.steps, 1), "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": args.precision, "data": "synthetic",
        "config": _config(args),
        "e2e": {"value": e2e, "unit": "tokens/s", "h2d_bytes_per_step": rec0.h2d_bytes,
                "d2h_bytes_per_step": rec0.d2h_bytes},
        "round": {"local_ms": rec0.local_ms, "aggregate_ms": rec0.aggregate_ms,
                  "host_stage_ms": rec0.host_ms, "mean_client_loss": rec0.mean_client_loss},
        "model_tflops": value * flops_per_token / 1e12,
        "mfu_vs_sustained": value * flops_per_token / 1e12 / world / bf16_sus,
        "clocks": clk.summary(),
    }
    if prof:
        ach = prof["gemm_flops"] / (prof["gemm_ms"] * 1e-3) / 1e12 if prof["gemm_ms"] else 0.0
        line["roofline"] = {"kernel": "gemm_tc (tcgen05, all client-step contractions)",
                            "bound": "tensor", "achieved": ach, "peak": bf16_sus,
                            "unit": "TFLOP/s", "frac": ach / bf16_sus,
                            "traffic": _gemm_traffic() if args.model == "125m" else None,
                            "traffic_unit": "DRAM bytes per launch (ncu, mean over one step's GEMMs)",
                            "peak_source": f"{peak_src} bf16 sustained"}
        line["kernel_ms_per_round"] = prof
        if prof["attn_ms"]:
            att = prof["attn_flops"] / (prof["attn_ms"] * 1e-3) / 1e12
            line["attention"] = {"kernel": "attn_*_tc (tcgen05; backward counted as 2.5x forward FLOPs)",
                                 "achieved_tflops": att, "frac_of_bf16_sustained": att / bf16_sus}
        line["gpu_launches"] = int(prof["launches"]) * args.steps
    if agg:
        line["aggregation"] = agg
    if world > 1:
        # the round boundary as run (NVLink peer-memory kernel, or NCCL above
        # PeerBoundary::fits): per-GPU wire bytes 2(G-1)/G * P * 4 over the
        # boundary's device time (RoundRecord.boundary_ms: the fused kernel once
        # every rank has arrived -- rank skew in the local phase excluded)
        P = model.param_count()
        wire = 2 * (world - 1) / world * P * 4
        line["boundary"] = {"ms_max_over_ranks": agg_ms_max, "wire_bytes_per_gpu": wire,
                            "busbw_gbs": wire / (agg_ms_max * 1e-3) / 1e9, "nvlink_gbs": 900.0,
                            "frac": wire / (agg_ms_max * 1e-3) / 1e9 / 900.0,
                            "path": _boundary_path(P)}
    if world == 1 and not args.no_cpu and args.model != "125m":
        # the f64 reference state of 1.3B / 7B exceeds host RAM
        line["cpu_baseline"] = {"value": None, "unit": "tokens/s", "cores": 0, "kind": "n/a",
                                "sample": f"reference CPU path not runnable at {args.model}"}
    elif world == 1 and not args.no_cpu:
        try:
            v, cores, kind, sample = cpu_sample(args.cpu_seq)
            line["cpu_baseline"] = {"value": v, "unit": "tokens/s", "cores": cores, "kind": kind,
                                    "sample": sample}
        except Exception as ex:  # pragma: no cover
            line["cpu_baseline"] = {"value": None, "unit": "tokens/s", "cores": 0,
                                    "kind": "unavailable", "sample": str(ex)[:200]}
    _emit(line)
    return 0


def main(argv=None):
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=3)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--tau", type=int, default=int(os.environ.get("PHOTON_BENCH_TAU", "64")))
    ap.add_argument("--batch", type=int, default=32)
    ap.add_argument("--precision", default="bf16", choices=["bf16", "f32"])
    ap.add_argument("--agg-k", type=int, default=8)
    ap.add_argument("--no-agg", action="store_true")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--cpu-seq", type=int, default=32)
    ap.add_argument("--model", default="125m", choices=sorted(MODELS),
                    help="125m is the contracted workload; 1.3b / 7b are SURVEY 8(d) configs 3-4")
    args = ap.parse_args(argv)
    if args.warmup < 3:
        args.warmup = 3
    if args.impl == "reference":
        return run_reference_arm(args)
    return run_ours(args)


if __name__ == "__main__":
    sys.exit(main())
