"""Development aid: per-phase instruction and stall attribution of an ncu source
page (--print-source sass), using an `nvdisasm -gi` listing of the same cubin.
Each SASS instruction is attributed to the first frame of its inline chain
(innermost first) whose bmc_kernel.cuh line falls in one of the phase ranges.

usage: python tools/ncu_phases.py DIS_gi.txt SRC.csv PER [KERNEL_SUBSTR [KERNEL.cuh]]
PER = divisor for instruction counts (e.g. B*(K+1) -> per instance-iteration)."""
import collections, csv, re, sys

# phases as (name, first-line anchor, last-line anchor) in bmc_kernel.cuh; resolved
# to line numbers at run time, so the attribution follows the current source
ANCHORS = [
    ("coll", "// Circular obstacles (coll_circ)", "// ------------------------------------------------------ temporal culling"),
    ("cull", "// ------------------------------------------------------ temporal culling", "// ---------------------------------------------------------------- phase B"),
    ("B.theta", "// ---------------------------------------------------------------- phase B", "// ---------------------------------------------------------------- phase D"),
    ("D2.mma", "  const double* __restrict__ P64 = pa.Pt64;", "#pragma unroll 1\n  for (int u = T - 1 - w; u < pa.rounds; u += T)"),
    ("D1.eval", "for (int u = T - 1 - w; u < pa.rounds; u += T)", "    BMC_SUB(pc, 12);"),
    ("D1.cullclk", "    BMC_SUB(pc, 12);", "    else {   // the plain loop"),
    ("D1.collcall", "    else {   // the plain loop", "    BMC_SUB(pc, 14);"),
    ("D1.U", "    BMC_SUB(pc, 14);", "  BMC_TICK(pc, 10);"),
    ("h.assembly", "  BMC_TICK(pc, 10);", "// ---------------------------------------------------------------- kernel"),
    ("prologue", "// ---------------------------------------------------------------- kernel", "    for (int it = -1; it < K; ++it) {"),
    ("A", "    for (int it = -1; it < K; ++it) {", "      // ---- B: heading target"),
    ("C", "      // ---- B: heading target", "      // ---- D: projections"),
    ("D.call", "      // ---- D: projections", "        // ---- E: multipliers"),
    ("E", "        // ---- E: multipliers", "    if (lp_pending) lampsi_step();"),
    ("epilogue", "    if (lp_pending) lampsi_step();", "size_t kernel_smem_bytes"),
]
RANGES = []


def resolve(src_path):
    lines = open(src_path).read().split("\n")
    def find(anchor, after=0):
        first = anchor.split("\n")[0]
        for i in range(after, len(lines)):
            if first in lines[i]:
                return i + 1
        raise ValueError(anchor)
    for name, a, b in ANCHORS:
        lo = find(a)
        hi = find(b, lo) - 1
        RANGES.append((name, lo, hi))


def frame_phase(chain):
    for f, ln in chain:
        if f.endswith("bmc_kernel.cuh"):
            for name, lo, hi in RANGES:
                if lo <= ln <= hi:
                    return name
    return "other"


def main():
    dis, src, per = sys.argv[1], sys.argv[2], float(sys.argv[3])
    ksel = sys.argv[4] if len(sys.argv) > 4 else "bmc_am_kernelILi3ELi2E"
    import os
    resolve(sys.argv[5] if len(sys.argv) > 5 else os.path.join(os.path.dirname(os.path.dirname(
        os.path.abspath(__file__))), "paper_2109_13030_b200", "csrc", "bmc_kernel.cuh"))
    insts, in_k, chain, fresh = [], False, [("?", 0)], True
    for l in open(dis):
        if l.strip().startswith(".section") and ".text." in l:
            in_k = ksel in l
            continue
        if not in_k:
            continue
        m = re.search(r'//## File "([^"]+)", line (\d+)(.*)', l)
        if m:   # one line per inline level, innermost first
            if fresh:
                chain, fresh = [], False
            chain.append((m.group(1), int(m.group(2))))
            continue
        m = re.match(r"\s*/\*([0-9a-f]{4,})\*/\s+(.*)", l)
        if m:
            fresh = True
            insts.append((frame_phase(chain), m.group(2).split(";")[0].strip()))
    rows = list(csv.reader(open(src)))
    hdr = rows[1]
    idx = {h: i for i, h in enumerate(hdr)}
    data = rows[2:]
    base = int(data[0][0], 16)
    stall_cols = [h for h in hdr if h.startswith("stall_") and "Not Issued" not in h]
    n_by, s_by = collections.Counter(), collections.Counter()
    st_by = collections.defaultdict(collections.Counter)
    op_by = collections.defaultdict(collections.Counter)
    for r in data:
        k = (int(r[0], 16) - base) // 16
        ph, op = insts[k] if k < len(insts) else ("?", "?")
        n = float(r[idx["Instructions Executed"]] or 0)
        n_by[ph] += n
        s_by[ph] += float(r[idx["Warp Stall Sampling (All Samples)"]] or 0)
        for c in stall_cols:
            st_by[ph][c[6:]] += float(r[idx[c]] or 0)
        mn = op.split()[0] if op else "?"
        if mn.startswith("@"):
            mn = op.split()[1]
        op_by[ph][mn.split(".")[0]] += n
    tn, ts = sum(n_by.values()), sum(s_by.values())
    print(f"total warp-inst per unit {tn / per:.1f}; stall samples {ts:.0f}")
    for ph, n in sorted(n_by.items(), key=lambda kv: -s_by[kv[0]]):
        top = ", ".join(f"{k} {100 * v / max(1, s_by[ph]):.0f}%" for k, v in st_by[ph].most_common(4))
        ops = ", ".join(f"{k} {v / per:.0f}" for k, v in op_by[ph].most_common(6))
        print(f"{ph:12s} inst {n / per:7.1f} ({100 * n / tn:4.1f}%)  stall {100 * s_by[ph] / ts:5.1f}%  [{top}]\n{'':14s}ops: {ops}")


if __name__ == "__main__":
    main()
