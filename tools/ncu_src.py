"""Summarise an `ncu --page source --csv --print-source sass` dump: stall-sample
share per instruction, with barrier waits / tcgen05 / TMA instructions always shown.
usage: ncu_src.py dump.csv [min_pct]"""
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
thr = float(sys.argv[2]) if len(sys.argv) > 2 else 0.8
hi = [i for i, r in enumerate(rows) if r and r[0] == "Address"][0]
h = rows[hi]
iS = h.index("Warp Stall Sampling (All Samples)")
iE = h.index("Instructions Executed")
data = [r for r in rows[hi + 1:] if len(r) == len(h) and r[0] != "Address"]
tot = sum(float(r[iS] or 0) for r in data) or 1.0
acc = 0.0
keys = ("TRYWAIT", "UTCBAR", "LDTM", "STTM", "BAR.SYNC", "EXIT", "UTMA")
for r in data:
    s = float(r[iS] or 0)
    acc += s
    ins = r[1]
    if s / tot * 100 > thr or (any(k in ins for k in keys) and int(r[iE] or 0) > 0):
        print(f"{r[0][-5:]} {s/tot*100:5.1f}% cum{acc/tot*100:5.1f}% ex={r[iE]:>9} {ins[:72]}")
