"""Summarise an ncu --csv launch list (gpu__time_duration / dram bytes): python scripts/ncu_kernels.py FILE [min_us]"""
import collections
import csv
import sys

lines = open(sys.argv[1]).read().splitlines()
min_us = float(sys.argv[2]) if len(sys.argv) > 2 else 10.0
start = [i for i, l in enumerate(lines) if l.startswith('"ID"')][0]
rows = list(csv.reader(lines[start:]))
hdr = rows[0]
ix = {h: i for i, h in enumerate(hdr)}
agg = collections.defaultdict(lambda: collections.defaultdict(list))
for r in rows[1:]:
    if len(r) != len(hdr):
        continue
    agg[r[ix["Kernel Name"]][:55]][r[ix["Metric Name"]]].append(float(r[ix["Metric Value"]].replace(",", "")))
for k, v in agg.items():
    t = v.get("gpu__time_duration.sum", [0.0])
    rd = v.get("dram__bytes_read.sum", [0.0])
    wr = v.get("dram__bytes_write.sum", [0.0])
    us = sum(t) / len(t) / 1e3
    if us >= min_us:
        gbs = (sum(rd) / len(rd) + sum(wr) / len(wr)) / (us * 1e3)
        print(f"{k:55s} n={len(t):4d} avg_us={us:8.1f} rd_MB={sum(rd)/len(rd)/1e6:8.1f} wr_MB={sum(wr)/len(wr)/1e6:8.1f} GB/s={gbs:7.0f}")
