"""Summarise an ncu --set full report + launch list into profiles/<tag>/SUMMARY.md (run in the build container).

    python profiles/summarize.py <tag> <full.ncu-rep> <launches.csv> [algorithmic_bytes_per_launch]
"""
import collections
import csv
import io
import os
import subprocess
import sys

KEYS = [
    "gpu__time_duration.sum", "sm__cycles_elapsed.avg.per_second", "dram__bytes_read.sum", "dram__bytes_write.sum",
    "dram__throughput.avg.pct_of_peak_sustained_elapsed", "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active",
    "sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active", "sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active",
    "smsp__issue_active.avg.pct_of_peak_sustained_active", "smsp__inst_executed.sum", "launch__registers_per_thread",
    "launch__occupancy_limit_registers", "sm__warps_active.avg.pct_of_peak_sustained_active",
    "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum.pct_of_peak_sustained_elapsed",
    "l1tex__t_requests_pipe_lsu_mem_local_op_ld.sum", "l1tex__t_requests_pipe_lsu_mem_local_op_st.sum",
    "smsp__sass_thread_inst_executed_op_dadd_pred_on.sum", "smsp__sass_thread_inst_executed_op_dmul_pred_on.sum",
    "smsp__sass_thread_inst_executed_op_dfma_pred_on.sum", "sm__inst_executed_pipe_tma.sum",
]


def raw_metrics(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr, units, vals = rows[0], rows[1], rows[2]
    return {h: (v, u) for h, u, v in zip(hdr, units, vals)}


def stalls(m):
    out = []
    for k, (v, _) in m.items():
        if k.startswith("smsp__average_warps_issue_stalled_") and k.endswith("_per_issue_active.ratio"):
            try:
                out.append((float(v), k[len("smsp__average_warps_issue_stalled_"):-len("_per_issue_active.ratio")]))
            except ValueError:
                pass
    return sorted(out, reverse=True)


def launches(path):
    rows = [r for r in csv.reader(open(path)) if len(r) > 5]
    hdr = rows[0]
    ki, mi, vi, ui = (hdr.index(x) for x in ("Kernel Name", "Metric Name", "Metric Value", "Metric Unit"))
    agg = collections.OrderedDict()
    for r in rows[1:]:
        if r[mi] != "gpu__time_duration.sum":
            continue
        v = float(r[vi].replace(",", ""))
        v = v * 1000 if r[ui] == "ms" else (v / 1000 if r[ui] == "ns" else v)
        agg.setdefault(r[ki].split("(")[0][:80], []).append(v)
    return agg


def inst_mix(rep, cells):
    out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                         capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    if len(rows) < 3:
        return None
    hdr, data = rows[1], rows[2:]
    isrc, iex = hdr.index("Source"), hdr.index("Instructions Executed")
    import re
    agg = collections.Counter()
    for r in data:
        m = re.match(r"(@!?U?P\w+\s+)?([A-Z0-9_]+)", r[isrc].strip())
        if m:
            agg[m.group(2)] += float(r[iex] or 0)
    return {k: v * 32 / cells for k, v in agg.items()}


def main():
    tag, rep, lcsv = sys.argv[1:4]
    alg = float(sys.argv[4]) if len(sys.argv) > 4 else None
    cells = float(sys.argv[5]) if len(sys.argv) > 5 else None
    os.makedirs(os.path.join("profiles", tag), exist_ok=True)
    m = raw_metrics(rep)
    lines = [f"# ncu summary `{tag}`", "", f"source: `{os.path.basename(rep)}` (ncu --set full, --clock-control none), "
             f"`{os.path.basename(lcsv)}` (launch list)", "", "## Fused kernel metrics (one launch)", "",
             "| metric | value | unit |", "|---|---|---|"]
    for k in KEYS:
        if k in m:
            lines.append(f"| {k} | {m[k][0]} | {m[k][1]} |")
    scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}

    def nbytes(key):   # each metric carries its own unit (read and write can differ)
        if key not in m:
            return None
        return float(m[key][0].replace(",", "")) * scale.get(m[key][1], 1)

    rd, wr = nbytes("dram__bytes_read.sum"), nbytes("dram__bytes_write.sum")
    if rd is not None and wr is not None and alg:
        lines += ["", f"DRAM traffic per launch: {(rd + wr) / 1e6:.1f} MB vs algorithmic "
                  f"{alg / 1e6:.1f} MB ({(rd + wr) / alg:.3f}x)"]
    lines += ["", "## Warp stall reasons (cycles per issued instruction)", "", "| reason | value |", "|---|---|"]
    for v, k in stalls(m)[:12]:
        lines.append(f"| {k} | {v:.3f} |")
    if cells:
        mix = inst_mix(rep, cells)
        if mix:
            tot = sum(mix.values())
            fp64 = sum(v for k, v in mix.items() if k in ("DADD", "DMUL", "DFMA", "DSETP"))
            lines += ["", f"## Instruction mix (thread instructions per cell update; {cells:.0f} cells per launch)", "",
                      f"total {tot:.1f}, FP64 {fp64:.1f}", "", "| opcode | per cell |", "|---|---|"]
            for k, v in sorted(mix.items(), key=lambda t: -t[1])[:20]:
                lines.append(f"| {k} | {v:.1f} |")
    agg = launches(lcsv)
    tot = sum(sum(v) for v in agg.values())
    lines += ["", "## Launch list (cold-cache, serialised; compare shares)", "",
              "| kernel | launches | avg us | share |", "|---|---|---|---|"]
    for k, v in agg.items():
        lines.append(f"| `{k}` | {len(v)} | {sum(v) / len(v):.2f} | {100 * sum(v) / tot:.1f}% |")
    with open(os.path.join("profiles", tag, "SUMMARY.md"), "w") as f:
        f.write("\n".join(lines) + "\n")
    print("\n".join(lines))


if __name__ == "__main__":
    main()
