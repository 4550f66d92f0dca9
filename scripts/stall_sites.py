"""Per-opcode instruction mix and the top stall sites of an ncu `--page source --csv` export.

    python scripts/stall_sites.py gpurun_out/<tag>_source.csv CELLS [TOP]
"""
import collections
import csv
import re
import sys

rows = list(csv.reader(open(sys.argv[1])))
cells = float(sys.argv[2])
top = int(sys.argv[3]) if len(sys.argv) > 3 else 25
hdr = rows[1]
data = rows[2:]
iS = hdr.index("Source")
iT = hdr.index("Thread Instructions Executed")
iW = hdr.index("Warp Stall Sampling (All Samples)")
cols = ["stall_barrier", "stall_wait", "stall_short_sb", "stall_long_sb", "stall_math", "stall_branch_resolving",
        "stall_mio", "stall_selected", "stall_not_selected", "stall_dispatch"]
ix = [hdr.index(c) for c in cols]
cnt, samp = collections.Counter(), collections.Counter()
reason = collections.Counter()
for r in data:
    m = re.match(r"(@!?U?P\w+\s+)?([A-Z][A-Z0-9]*(\.[A-Z0-9]+)*)", r[iS].strip())
    if not m:
        continue
    cnt[m.group(2)] += int(r[iT])
    samp[m.group(2)] += int(r[iW])
    for c, j in zip(cols, ix):
        reason[c] += int(r[j] or 0)
tot = sum(int(r[iW]) for r in data)
print(f"instructions per cell {sum(cnt.values()) / cells:.1f}; stall samples {tot}")
print("reasons:", ", ".join(f"{c[6:]} {100.0 * v / tot:.1f}%" for c, v in reason.most_common()))
for op, c in cnt.most_common(20):
    print(f"  {op:28s} {c / cells:7.2f}/cell  samples {samp[op]}")
print("top stall sites:")
for i in sorted(sorted(range(len(data)), key=lambda i: -int(data[i][iW]))[:top]):
    r = data[i]
    why = max(zip(cols, ix), key=lambda t: int(r[t[1]] or 0))[0][6:]
    print(f"  {i:5d} {int(r[iW]):5d} {why:15s} {r[iS].strip()[:70]}")
