"""Per-class roofline table of one 125M client step from the round-2 ncu CSVs
(tools/capture_r02.sh): every tcgen05 GEMM launch of the step is matched to
its contraction by launch order (engine.cu's static schedule), so each class
gets its algorithmic FLOPs and bytes next to the measured time, DRAM bytes
and tensor-pipe utilisation; attention and memory-bound kernels likewise.

    python tools/step_table.py gpurun_out profiles/r02_step
        -> profiles/r02_step.txt (tables) and profiles/r02_step.json
"""
import collections
import csv
import json
import os
import sys

L, d, H, V, S, B = 12, 768, 12, 50368, 2048, 32
M, hid, dh = B * S, 4 * d, d // H
UNIT = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "nsecond": 1e-3, "usecond": 1.0,
        "msecond": 1e3, "ns": 1e-3, "us": 1.0, "ms": 1e3, "%": 1, "inst": 1, "cycle": 1,
        "hz": 1, "Khz": 1e3, "Mhz": 1e6, "Ghz": 1e9, "Hz": 1, "KHz": 1e3, "MHz": 1e6, "GHz": 1e9,
        "cycle/second": 1, "cycle/nsecond": 1e9, "cycle/usecond": 1e6}


def launches(path):
    """ncu --csv log -> [ {kernel, metric: value} ] in launch order."""
    by_id = collections.OrderedDict()
    with open(path) as f:
        lines = [l for l in f if l.startswith('"')]
    for r in csv.DictReader(lines):
        k = by_id.setdefault(r["ID"], {"kernel": r["Kernel Name"].split("(")[0].replace("void ", ""),
                                        "grid": r["Grid Size"]})
        try:
            v = float(r["Metric Value"].replace(",", ""))
        except ValueError:
            continue
        k[r["Metric Name"]] = v * UNIT.get(r["Metric Unit"], 1)
    return list(by_id.values())


def gemm_schedule():
    """(class, M, N, K, bytes) per GEMM launch of one step, in launch order.
    bytes: bf16 operands read once, output written once (+ epilogue inputs)."""
    def g(cls, m, n, k, out_bytes=2, extra=0):
        return (cls, m, n, k, 2 * m * k + 2 * k * n + out_bytes * m * n + extra)
    s = []
    for _ in range(L):
        s += [g("fwd qkv", M, d, d)] * 3
        s.append(g("fwd wo (+resid, fp32 out)", M, d, d, 4, 4 * M * d))
        s.append(g("fwd w1 (GELU, 2 outputs)", M, hid, d, 4))
        s.append(g("fwd w2 (+resid, fp32 out)", M, d, hid, 4, 4 * M * d))
    s.append(g("fwd head", M, V, d))
    s.append(g("bwd head dX", M, d, V, 4))
    s.append(g("bwd head dW", d, V, M, 4))
    for _ in range(L):
        s.append(g("bwd w2 dX (GELU')", M, hid, d, 2, 2 * M * hid))
        s.append(g("bwd dW d x 4d / 4d x d", hid, d, M, 4))
        s.append(g("bwd w1 dX", M, d, hid, 4))
        s.append(g("bwd dW d x 4d / 4d x d", d, hid, M, 4))
        s.append(g("bwd wo dX", M, d, d))
        s.append(g("bwd dW d x d", d, d, M, 4))
        s.append(g("bwd qkv dX (K-concat)", M, d, 3 * d, 4))
        s += [g("bwd dW d x d", d, d, M, 4)] * 3
    return s


def main(src, stem):
    out, js = [], {}
    gl = launches(os.path.join(src, "r02_gemm_step.csv"))
    sched = gemm_schedule()
    assert len(gl) == len(sched), (len(gl), len(sched))
    cls = collections.OrderedDict()
    for k, (c, m, n, kk, nbytes) in zip(gl, sched):
        e = cls.setdefault(c, collections.defaultdict(float))
        e["n"] += 1
        e["us"] += k["gpu__time_duration.sum"]
        e["flop"] += 2.0 * m * n * kk
        e["alg_bytes"] += nbytes
        e["dram"] += k["dram__bytes_read.sum"] + k["dram__bytes_write.sum"]
        e["tensor_pct_x_us"] += k["sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active"] * k["gpu__time_duration.sum"]
        e["hmma_pct_x_us"] += k["sm__pipe_tensor_subpipe_hmma_cycles_active.avg.pct_of_peak_sustained_active"] * k["gpu__time_duration.sum"]
        e["clk_x_us"] += k["sm__cycles_elapsed.avg.per_second"] * k["gpu__time_duration.sum"]
    tot = collections.defaultdict(float)
    out.append("GEMM classes, one steady-state step (195 tcgen05 launches; ncu, serialised,"
               " --clock-control none)")
    out.append("class | launches | ms | TFLOP/s | tensor pipe % (time-weighted) | "
               "DRAM GB | algorithmic GB | DRAM / algorithmic | mean SM MHz")
    for c, e in cls.items():
        for key in e:
            tot[key] += e[key]
        row = {"launches": int(e["n"]), "ms": e["us"] / 1e3,
               "tflops": e["flop"] / (e["us"] * 1e-6) / 1e12,
               "tensor_pipe_pct": e["tensor_pct_x_us"] / e["us"],
               "hmma_subpipe_pct": e["hmma_pct_x_us"] / e["us"],
               "dram_gb": e["dram"] / 1e9, "alg_gb": e["alg_bytes"] / 1e9,
               "dram_over_alg": e["dram"] / e["alg_bytes"],
               "sm_mhz": e["clk_x_us"] / e["us"] / 1e6}
        js[c] = row
        out.append(f"{c} | {row['launches']} | {row['ms']:.3f} | {row['tflops']:.0f} | "
                   f"{row['tensor_pipe_pct']:.1f} | {row['dram_gb']:.2f} | {row['alg_gb']:.2f} | "
                   f"{row['dram_over_alg']:.2f} | {row['sm_mhz']:.0f}")
    allrow = {"launches": int(tot["n"]), "ms": tot["us"] / 1e3,
              "tflops": tot["flop"] / (tot["us"] * 1e-6) / 1e12,
              "tensor_pipe_pct": tot["tensor_pct_x_us"] / tot["us"],
              "dram_gb": tot["dram"] / 1e9, "alg_gb": tot["alg_bytes"] / 1e9,
              "dram_bytes_per_launch": tot["dram"] / tot["n"],
              "alg_bytes_per_launch": tot["alg_bytes"] / tot["n"],
              "flop": tot["flop"], "sm_mhz": tot["clk_x_us"] / tot["us"] / 1e6}
    js["ALL GEMMs"] = allrow
    out.append(f"ALL | {allrow['launches']} | {allrow['ms']:.3f} | {allrow['tflops']:.0f} | "
               f"{allrow['tensor_pipe_pct']:.1f} | {allrow['dram_gb']:.2f} | {allrow['alg_gb']:.2f}"
               f" | {tot['dram'] / tot['alg_bytes']:.2f} | {allrow['sm_mhz']:.0f}")
    out.append(f"mean DRAM bytes per GEMM launch (bench.py roofline.traffic): "
               f"{allrow['dram_bytes_per_launch']:.4g}; algorithmic {allrow['alg_bytes_per_launch']:.4g}")

    # attention: fwd FLOPs 4*B*H*dh*S(S+1)/2 per layer, backward 2.5x (the fused pass, or
    # 1.25x for each of the two recomputing passes)
    p = os.path.join(src, "r02_attn_step.csv")
    if os.path.exists(p):
        at = collections.OrderedDict()
        fwd = 4.0 * B * H * dh * S * (S + 1) / 2
        for k in launches(p):
            name = k["kernel"].split("<")[0].split("::")[-1]
            e = at.setdefault(name, collections.defaultdict(float))
            t = k["gpu__time_duration.sum"]
            e["n"] += 1
            e["us"] += t
            for m_, key in (("sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active", "tensor"),
                            ("sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active", "fma"),
                            ("sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_active", "alu")):
                e[key] += k.get(m_, 0.0) * t
            e["xu_inst"] += k.get("sm__inst_executed_pipe_xu.sum", 0.0)
            e["dram"] += k["dram__bytes_read.sum"] + k["dram__bytes_write.sum"]
            e["clk"] += k["sm__cycles_elapsed.avg.per_second"] * t
        out.append("")
        out.append("attention kernels, one step (12 layers)")
        out.append("kernel | launches | ms | tensor pipe % | FMA pipe % | ALU pipe % | "
                   "XU (MUFU) warp-inst per launch | DRAM GB | TFLOP/s (fwd convention)")
        for name, e in at.items():
            fl = (fwd * e["n"] if "fwd" in name else
                  2.5 * fwd * e["n"] if "fused" in name else
                  1.25 * fwd * e["n"] if ("dkdv" in name or "dq" in name) else 0.0)
            row = {"launches": int(e["n"]), "ms": e["us"] / 1e3,
                   "tensor_pipe_pct": e["tensor"] / e["us"], "fma_pipe_pct": e["fma"] / e["us"],
                   "alu_pipe_pct": e["alu"] / e["us"], "xu_inst_per_launch": e["xu_inst"] / e["n"],
                   "dram_gb": e["dram"] / 1e9,
                   "tflops": fl / (e["us"] * 1e-6) / 1e12 if fl else None,
                   "sm_mhz": e["clk"] / e["us"] / 1e6}
            js["attn:" + name] = row
            out.append(f"{name} | {row['launches']} | {row['ms']:.3f} | {row['tensor_pipe_pct']:.1f} | "
                       f"{row['fma_pipe_pct']:.1f} | {row['alu_pipe_pct']:.1f} | "
                       f"{row['xu_inst_per_launch']:.3g} | {row['dram_gb']:.2f} | "
                       f"{row['tflops'] if row['tflops'] is None else round(row['tflops'])}")

    p = os.path.join(src, "r02_other_step.csv")
    if os.path.exists(p):
        ot = collections.OrderedDict()
        ls = launches(p)
        half = ls[len(ls) // 2:]  # second round's launches
        for k in half:
            name = k["kernel"].split("<")[0].split("::")[-1]
            e = ot.setdefault(name, collections.defaultdict(float))
            e["n"] += 1
            e["us"] += k["gpu__time_duration.sum"]
            e["dram"] += k["dram__bytes_read.sum"] + k["dram__bytes_write.sum"]
        out.append("")
        out.append("memory-bound kernels, one step (second round's launches)")
        out.append("kernel | launches | ms | DRAM GB | DRAM GB/s")
        for name, e in sorted(ot.items(), key=lambda kv: -kv[1]["us"]):
            row = {"launches": int(e["n"]), "ms": e["us"] / 1e3, "dram_gb": e["dram"] / 1e9,
                   "dram_gbs": e["dram"] / (e["us"] * 1e-6) / 1e9}
            js["mem:" + name] = row
            out.append(f"{name} | {row['launches']} | {row['ms']:.3f} | {row['dram_gb']:.2f} | "
                       f"{row['dram_gbs']:.0f}")
    with open(stem + ".txt", "w") as f:
        f.write("\n".join(out) + "\n")
    with open(stem + ".json", "w") as f:
        json.dump(js, f, indent=1)
    print("\n".join(out))


if __name__ == "__main__":
    main(sys.argv[1], sys.argv[2])
