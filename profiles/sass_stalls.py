"""Summarise an ncu source-page CSV (--page source --csv --print-source sass):
stall samples by reason and by opcode, and the hottest instructions.
    python profiles/sass_stalls.py sass.csv [top]
"""
import collections
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
top = int(sys.argv[2]) if len(sys.argv) > 2 else 40
hdr = rows[1]
ix = {h: i for i, h in enumerate(hdr)}
reasons = [h for h in hdr if h.startswith("stall_") and "Not Issued" not in h]
body = [r for r in rows[2:] if len(r) == len(hdr)]
tot = collections.Counter()
by_op = collections.defaultdict(collections.Counter)
samples = 0
for r in body:
    op = r[1].strip().split()[0] if r[1].strip() else "?"
    if op.startswith("@"):
        op = r[1].strip().split()[1]
    op = op.split(".")[0]
    for h in reasons:
        v = int(r[ix[h]] or 0)
        tot[h] += v
        by_op[op][h] += v
        samples += v
print(f"total samples {samples}")
for h, v in tot.most_common():
    if v:
        print(f"  {h:24s} {v:8d} {100*v/samples:5.1f}%")
print("\nby opcode (samples, top reasons)")
ops = sorted(by_op.items(), key=lambda kv: -sum(kv[1].values()))
for op, c in ops[:20]:
    s = sum(c.values())
    print(f"  {op:10s} {s:8d} {100*s/samples:5.1f}%  " + ", ".join(f"{k[6:]}={v}" for k, v in c.most_common(3)))
print("\nhottest instructions")
hot = sorted(body, key=lambda r: -int(r[ix["Warp Stall Sampling (All Samples)"]] or 0))[:top]
for r in hot:
    c = {h[6:]: int(r[ix[h]] or 0) for h in reasons}
    best = sorted(c.items(), key=lambda kv: -kv[1])[:2]
    print(f"  {r[0][-5:]} {r[ix['Warp Stall Sampling (All Samples)']]:>6s} {r[1].strip()[:60]:60s} {best}")
