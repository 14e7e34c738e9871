"""Summarise an ncu report into profiles/<name>.md (key metrics, stall reasons,
instruction mix, hottest source lines).  usage: ncu_summary.py REPORT NAME [OBJ]"""
import collections, csv, io, os, re, subprocess, sys

rep, name = sys.argv[1], sys.argv[2]
obj = sys.argv[3] if len(sys.argv) > 3 else None
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

def ncu(*args):
    return subprocess.run(["ncu", "-i", rep, *args], capture_output=True, text=True).stdout

raw = list(csv.reader(io.StringIO(ncu("--page", "raw", "--csv"))))
d = dict(zip(raw[0], raw[2])) if len(raw) > 2 else {}
keys = ["gpu__time_duration.sum", "smsp__inst_executed.sum", "smsp__issue_active.avg.pct_of_peak_sustained_active",
        "smsp__warps_active.avg.per_cycle_active", "smsp__warps_eligible.avg.per_cycle_active",
        "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active",
        "sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active",
        "dram__bytes_read.sum", "dram__bytes_write.sum", "launch__registers_per_thread",
        "launch__grid_size", "launch__block_size", "launch__occupancy_limit_registers",
        "launch__occupancy_limit_shared_mem", "sm__warps_active.avg.pct_of_peak_sustained_active",
        "sm__cycles_elapsed.avg.per_second"]
lines = [f"# ncu summary: {name}", "", f"report: `{os.path.basename(rep)}`", "", "| metric | value |", "|---|---|"]
for k in keys:
    lines.append(f"| {k} | {d.get(k)} |")
st = [(k[34:-23], float(v)) for k, v in d.items()
      if k.startswith("smsp__average_warps_issue_stalled") and k.endswith("_per_issue_active.ratio") and v not in ("", "n/a")]
st.sort(key=lambda x: -x[1])
lines += ["", "Stall reasons (cycles per issued instruction):", ""]
lines += [f"- {k}: {v:.2f}" for k, v in st if v > 0.02]
sass = list(csv.reader(io.StringIO(ncu("--page", "source", "--csv", "--print-source", "sass"))))
if len(sass) > 2:
    hdr = sass[1]; idx = {h: i for i, h in enumerate(hdr)}
    ops = collections.Counter(); tot = 0
    for r in sass[2:]:
        n = float(r[idx["Instructions Executed"]] or 0)
        s = re.sub(r"^@!?U?P\w+\s+", "", r[idx["Source"]].strip())
        ops[s.split()[0] if s else "?"] += n; tot += n
    lines += ["", f"Instruction mix (warp-level, total {tot:.4g}):", "", "| opcode | share |", "|---|---|"]
    lines += [f"| {op} | {100 * n / tot:.1f}% |" for op, n in ops.most_common(20)]
open(os.path.join(ROOT, "profiles", f"{name}.md"), "w").write("\n".join(lines) + "\n")
print("\n".join(lines[:40]))
