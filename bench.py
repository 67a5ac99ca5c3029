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

  --impl reference  the reference's own FederationRunner (oracle/_ref, built from
         /root/reference sources) on the host cores: at --model small the
         identical round (same_config), at 125m a stated reduced-context sample.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--model M] [--impl reference]
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
# the hetero4 decoder (configs/hetero4.cfg:15-21, the one
# config the reference CPU path runs in full), Photon 125M / 1.3B / 7B
MODELS = {"small": ((1, 32, 2, 4, 64, 16), "hetero4 decoder (config 1)", "17,440"),
          "125m": (MODEL_125M, "Photon-125M", "164.04M"),
          "1.3b": ((24, 2048, 16, 4, 50368, 2048), "Photon-1.3B", "1,419.15M"),
          "7b": ((32, 4096, 32, 4, 50368, 2048), "Photon-7B", "6,865.22M")}
# per model: (tau, B, clients per GPU, LrSchedule(eta_max, warmup, decay, alpha))
RUN = {"small": (16, 4, 2, (2e-3, 16, 160, 0.1)),   # hetero4.cfg:37-42, 2 clients
       "125m": (64, 32, 1, (6e-4, 64, 1024, 0.1)),
       "1.3b": (64, 32, 1, (6e-4, 64, 1024, 0.1)),
       "7b": (64, 32, 1, (6e-4, 64, 1024, 0.1))}
# the reference CPU arm at 125M: the full S = 2048 step costs ~15 min of f64 per
# client, so each client of its FederationRunner round runs the same
# architecture at a reduced sequence length (stated in its config)
REF_SEQ_125M = 32
MEASURED_PEAKS = os.path.join(ROOT, "MEASURED_PEAKS.json")
METRIC = "tokens/s/round at 1-8 B200 (125M); FedAvg aggregate GB/s vs roofline"


NCU_STEP = os.path.join(ROOT, "profiles", "r02d_step.json")


def _gemm_ncu():
    """ncu evidence for the roofline kernel class: mean DRAM bytes (read + write)
    per tcgen05 GEMM launch over ALL 195 GEMM launches of one 125M client step,
    their algorithmic bytes, and the time-weighted tensor-pipe utilisation
    (tools/capture_r02d.sh -> tools/step_table.py -> profiles/r02d_step.json)."""
    try:
        with open(NCU_STEP) as f:
            g = json.load(f)["ALL GEMMs"]
        return {"traffic": g["dram_bytes_per_launch"],
                "algorithmic_bytes_per_launch": g["alg_bytes_per_launch"],
                "tensor_pipe_pct_ncu": g["tensor_pipe_pct"], "launches_per_step": g["launches"]}
    except Exception:
        return {"traffic": None}


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
# CPU baseline: the reference's own FederationRunner (oracle/_ref) on host cores
# ---------------------------------------------------------------------------
def _cpu_model() -> str:
    try:
        with open("/proc/cpuinfo") as f:
            return next(l.split(":", 1)[1].strip() for l in f if l.startswith("model name"))
    except Exception:
        return "unknown"


def _cpu_threads(per_client_gb: float = 9.0):
    n = os.cpu_count() or 1
    try:
        with open("/proc/meminfo") as f:
            avail_kb = next(int(l.split()[1]) for l in f if l.startswith("MemAvailable"))
        by_mem = max(1, int(avail_kb / 1024 / 1024 / per_client_gb))
    except Exception:
        by_mem = 4
    return max(1, min(n, by_mem, 64))


def ref_rounds(model: str, gpus: int, rounds: int, warmup: int = 1):
    """The reference's FederationRunner::run_round (aggregator.cpp:93-220) on the
    host: n_threads = min(K, nproc), eval_every = 0, no checkpoints; corpus,
    partition, streams and init exactly as our arm builds them.  Returns
    (tokens/s from the median round, per-round seconds, description dict).

    small: the identical workload our arm runs (K = 2 per GPU, tau 16, B 4).
    125m:  K = host threads clients, tau = 1, B = 1 at S = REF_SEQ_125M --
           the same architecture with a shorter context (labelled as such)."""
    from oracle import ModelCfg, ServerCfg, TrainCfg, load_oracle, load_reference

    shape = list(MODELS[model][0])
    tau, B, per_gpu, sched = RUN[model]
    if model == "small":
        K = per_gpu * gpus
        threads = min(K, os.cpu_count() or 1)
    else:
        shape[5] = REF_SEQ_125M
        tau, B = 1, 1
        K = threads = _cpu_threads()
    mc = ModelCfg(*shape)
    S, V = shape[5], shape[4]
    t = TrainCfg(eta_max=sched[0], warmup_steps=sched[1], decay_steps=sched[2], alpha=sched[3],
                 local_steps=tau, batch_size=B)
    n_tok = K * tau * B * (S + 1) * (rounds + warmup) + S + 1
    ref = load_reference()
    kind = "reference"
    if ref is None:
        raise RuntimeError("oracle/_ref (the reference built from its own sources) is missing")
    theta0 = load_oracle().init_params(mc, 1)
    _, _, _, secs = ref.run_rounds(mc, t, ServerCfg(1, 0.1, 0.9, 1), 0, "web", n_tok, 7, K, K,
                                   rounds + warmup, 42, 2, threads, theta0)
    timed = list(secs[warmup:])
    tokens = K * tau * B * S
    L, d, H, e = shape[:4]
    desc = {"model": f"L{L} d{d} H{H} e{e} V{V} S{S}", "clients": K, "local_steps": tau,
            "batch": B, "seq_len": S, "tokens_per_round": tokens, "threads": threads,
            "nproc": os.cpu_count(), "cpu_model": _cpu_model(), "kind": kind,
            "round_seconds": timed, "warmup_rounds": warmup,
            "how": "FederationRunner::run_round, eval_every=0, n_threads=min(K, nproc); "
                   "median of the timed rounds"}
    return tokens / statistics.median(timed), timed, desc


def run_reference_arm(args):
    rank, world, local = _dist_setup(args.gpus)
    if rank != 0:
        return 0
    # one FederationRunner session: W warm-up rounds, then K timed rounds
    t0 = time.perf_counter()
    # at 125m every round is ~10-30 s of f64 work per host thread: one warm-up
    # round, so the arm ends within minutes
    warm = args.warmup if args.model == "small" else 1
    value, secs, desc = ref_rounds(args.model, args.gpus, args.steps, warmup=warm)
    wall = time.perf_counter() - t0
    same = args.model == "small"
    cfg = dict(_config(args), precision="f64 (the reference's own arithmetic)",
               clients=desc["clients"], local_steps=desc["local_steps"], batch=desc["batch"],
               seq_len=desc["seq_len"], model=desc["model"],
               global_batch=desc["clients"] * desc["batch"], threads=desc["threads"],
               nproc=desc["nproc"], cpu_model=desc["cpu_model"], same_config=same)
    if not same:
        cfg["sample_of"] = _config(args)["model"]
    sample = (f"{desc['clients']} reference clients x tau={desc['local_steps']} x "
              f"B={desc['batch']} x S={desc['seq_len']} per round, {desc['model']}, "
              f"{desc['threads']} host threads ({desc['cpu_model']}, nproc {desc['nproc']}); "
              f"median of {len(secs)} FederationRunner rounds after {warm} warm-up")
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": "tokens/s",
        "n_gpus": args.gpus, "steps": args.steps, "warmup": warm,
        "ms_per_step": 1000.0 * statistics.median(secs), "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": cfg,
        "cpu_baseline": {"value": value, "unit": "tokens/s", "cores": desc["threads"],
                         "kind": desc["kind"], "sample": sample},
        "e2e": {"value": value, "unit": "tokens/s", "h2d_bytes_per_step": 0,
                "d2h_bytes_per_step": 0},
        "round_seconds": secs, "wall_s": wall,
    }
    _emit(line)
    return 0


def _config(args):
    shape, name, params = MODELS[args.model]
    L, d, H, e, V, S = shape
    per_gpu = args.clients_per_gpu
    server = "nesterov eta=0.1 mu=0.9"
    return {"workload": f"{name} federated round (reference architecture, {params} params)",
            "model": f"L{L} d{d} H{H} e{e} V{V} S{S}", "clients": args.gpus * per_gpu,
            "clients_per_gpu": per_gpu, "local_steps": args.tau, "batch": args.batch,
            "seq_len": S, "global_batch": args.gpus * per_gpu * args.batch,
            "server_opt": server, "parallelism": f"fed{args.gpus}", "precision": args.precision,
            "micro_batch": args.micro_batch or args.batch,
            "l2": "inputs larger than L2 (weights+activations >> 126 MB)"
            if args.model != "small" else "model and batch fit in L2 (config 1 is tiny)"}


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
    per_gpu = args.clients_per_gpu
    K = world * per_gpu  # weak scaling: clients per GPU fixed
    rounds = args.warmup + args.steps + 1
    tau, B = args.tau, args.batch
    sched = RUN[args.model][3]
    # corpus: one epoch per client per round of tau*B blocks of S+1 tokens
    n_tok = K * tau * B * (S + 1) + S + 1
    corpus = F.generate_corpus("web", n_tok, 7, V)
    plan = F.partition_iid(corpus, K, S, 7)
    theta0 = F.TransformerModel(model).init_params(1)
    local_cfg = F.LocalTrainConfig(model=model, schedule=F.LrSchedule(*sched),
                                   local_steps=tau, batch_size=B)
    server = F.ServerOptConfig(1, 0.1, 0.9, True)
    nccl_id = _bcast_bytes(F.nccl_unique_id() if rank == 0 else b"", world, local) \
        if world > 1 else None
    runner = F.FederationRunner(F.FederationConfig(K, K, rounds, F.Topology.kRingAllReduce, 42),
                                local_cfg, server, plan, theta0, device=local,
                                precision=args.precision, rank=rank, world=world,
                                nccl_id=nccl_id, micro_batch=args.micro_batch)
    for _ in range(args.warmup):
        runner.run_round()

    # ---- timed region: K rounds, barrier + sync on both sides
    import torch

    torch.cuda.synchronize(local)
    _barrier(world)
    dev_ms, recs = 0.0, []
    lib = A.lib()
    n_launch0 = lib.photon_launch_count()
    with ClockSampler(local) as clk:
        t0 = time.perf_counter()
        for _ in range(args.steps):
            rec = runner.run_round()
            recs.append(rec)
            dev_ms += rec.round_ms
        torch.cuda.synchronize(local)
        wall = time.perf_counter() - t0
    n_launch = lib.photon_launch_count() - n_launch0
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
                "attn_launches": times[6], "spans": times[7]}

    agg = None
    if rank == 0 and not args.no_agg and args.model != "small":
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
        ncu = _gemm_ncu() if args.model == "125m" else {"traffic": None}
        line["roofline"] = dict({"kernel": "gemm_tc (tcgen05, all client-step contractions)",
                                 "bound": "tensor", "achieved": ach, "peak": bf16_sus,
                                 "unit": "TFLOP/s", "frac": ach / bf16_sus},
                                **ncu, traffic_unit="DRAM bytes per launch (ncu, mean over all "
                                                    "195 GEMM launches of one step)",
                                peak_source=f"{peak_src} bf16 sustained")
        line["kernel_ms_per_round"] = prof
        if prof["attn_ms"]:
            att = prof["attn_flops"] / (prof["attn_ms"] * 1e-3) / 1e12
            line["attention"] = {"kernel": "attn_*_tc (tcgen05; backward counted as 2.5x forward FLOPs)",
                                 "achieved_tflops": att, "frac_of_bf16_sustained": att / bf16_sus}
    # our kernels launched in the timed region on this rank (every launch site +
    # the kernel nodes of each CUDA-graph replay)
    line["gpu_launches"] = int(n_launch)
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
    if world == 1 and not args.no_cpu and args.model not in ("125m", "small"):
        # the f64 reference state of 1.3B / 7B exceeds host RAM
        line["cpu_baseline"] = {"value": None, "unit": "tokens/s", "cores": 0, "kind": "n/a",
                                "sample": f"reference CPU path not runnable at {args.model}"}
    elif world == 1 and not args.no_cpu:
        try:
            # one bounded FederationRunner round of the reference (no warm-up:
            # keeps the default bench within minutes; --impl reference is the
            # warmed, median-of-rounds measurement)
            v, secs, desc = ref_rounds(args.model, 1, 1, warmup=0)
            line["cpu_baseline"] = {
                "value": v, "unit": "tokens/s", "cores": desc["threads"], "kind": desc["kind"],
                "sample": f"{desc['clients']} reference clients x tau={desc['local_steps']} x "
                          f"B={desc['batch']} x S={desc['seq_len']}, {desc['model']}, one "
                          f"FederationRunner round on {desc['threads']} host threads "
                          f"({desc['cpu_model']}, nproc {desc['nproc']})",
                "same_config": args.model == "small"}
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
    ap.add_argument("--tau", type=int, default=None, help="local steps (default per model)")
    ap.add_argument("--batch", type=int, default=None, help="local batch (default per model)")
    ap.add_argument("--micro-batch", type=int, default=None,
                    help="activation rows per micro-batch (default: the whole local batch)")
    ap.add_argument("--clients-per-gpu", type=int, default=None,
                    help="sampled clients trained per GPU each round (default per model)")
    ap.add_argument("--precision", default="bf16", choices=["bf16", "f32"])
    ap.add_argument("--agg-k", type=int, default=8)
    ap.add_argument("--no-agg", action="store_true")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--model", default="125m", choices=sorted(MODELS),
                    help="125m is the contracted workload; small / 1.3b / 7b are SURVEY "
                         "8(d) configs 1, 3, 4 (small: both arms run the identical round)")
    args = ap.parse_args(argv)
    if args.tau is None:
        args.tau = int(os.environ.get("PHOTON_BENCH_TAU", RUN[args.model][0]))
    if args.batch is None:
        args.batch = RUN[args.model][1]
    if args.clients_per_gpu is None:
        args.clients_per_gpu = RUN[args.model][2]
    if args.warmup < 3:
        args.warmup = 3
    if args.impl == "reference":
        return run_reference_arm(args)
    return run_ours(args)


if __name__ == "__main__":
    sys.exit(main())
