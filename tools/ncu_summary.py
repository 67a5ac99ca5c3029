"""Summarise an `ncu --set full` report: per launch duration, DRAM bytes, tensor
pipe and TMEM activity; per kernel averages as JSON (bench.py reads the
`traffic` of its roofline kernel from that JSON).

    python tools/ncu_summary.py gpurun_out/step_full.ncu-rep profiles/r01_ncu_step_full
        -> profiles/r01_ncu_step_full.txt, profiles/r01_ncu_step_full.json
"""
import collections
import csv
import io
import json
import subprocess
import sys

METRICS = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
           "sm__inst_executed_pipe_tmem.avg.pct_of_peak_sustained_active",
           "sm__throughput.avg.pct_of_peak_sustained_elapsed",
           "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
           "launch__registers_per_thread", "sm__cycles_elapsed.avg.per_second"]
UNIT = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "ns": 1e-3, "us": 1.0, "ms": 1e3,
        "nsecond": 1e-3, "usecond": 1.0, "msecond": 1e3, "Hz": 1, "KHz": 1e3, "MHz": 1e6,
        "GHz": 1e9}


def rows(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"],
                         capture_output=True, text=True, check=True).stdout
    rs = list(csv.reader(io.StringIO(out)))
    # the full set prefixes some names with their section ("TPC.TriageCompute.")
    hdr = [h.split(".", 2)[-1] if h.count(".") > 2 and h.split(".")[0].isupper() else h for h in rs[0]]
    units = rs[1]
    for r in rs[2:]:
        if len(r) != len(hdr):
            continue
        d = {"kernel": r[hdr.index("Kernel Name")].split("(")[0].replace("void ", "")}
        d["grid"], d["block"] = r[hdr.index("Grid Size")], r[hdr.index("Block Size")]
        for m in METRICS:
            if m in hdr:
                i = hdr.index(m)
                try:
                    v = float(r[i].replace(",", ""))
                except ValueError:
                    v = float("nan")
                d[m] = v * UNIT.get(units[i], 1)
        yield d


def main(rep, stem):
    data = list(rows(rep))
    lines = ["kernel | grid | us | DRAM rd MB | DRAM wr MB | DRAM GB/s | tmem % | SM % | regs"]
    per = collections.defaultdict(list)
    for d in data:
        us = d["gpu__time_duration.sum"]
        rd, wr = d["dram__bytes_read.sum"], d["dram__bytes_write.sum"]
        lines.append(f"{d['kernel'][:60]} | {d['grid']} | {us:.1f} | {rd/1e6:.1f} | {wr/1e6:.1f} | "
                     f"{(rd+wr)/us/1e3:.0f} | "
                     f"{d.get('sm__inst_executed_pipe_tmem.avg.pct_of_peak_sustained_active', float('nan')):.1f} | "
                     f"{d.get('sm__throughput.avg.pct_of_peak_sustained_elapsed', float('nan')):.1f} | "
                     f"{d.get('launch__registers_per_thread', float('nan')):.0f}")
        per[d["kernel"]].append(d)
    summary = {}
    for k, ds in per.items():
        n = len(ds)
        summary[k] = {"launches": n,
                      "us_per_launch": sum(d["gpu__time_duration.sum"] for d in ds) / n,
                      "dram_bytes_per_launch": sum(d["dram__bytes_read.sum"] + d["dram__bytes_write.sum"]
                                                   for d in ds) / n}
    open(stem + ".txt", "w").write("\n".join(lines) + "\n")
    json.dump({"report": rep, "kernels": summary}, open(stem + ".json", "w"), indent=1)
    print("\n".join(lines))


if __name__ == "__main__":
    main(sys.argv[1], sys.argv[2])
