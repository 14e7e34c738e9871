"""Development aid: per-phase instruction and stall attribution of an ncu source
page (--print-source sass), using an `nvdisasm -gi` listing of the same cubin.
Each SASS instruction is attributed to the first frame of its inline chain
(innermost first) whose bmc_kernel.cuh line falls in one of the phase ranges.

usage: python tools/ncu_phases.py DIS_gi.txt SRC.csv PER [KERNEL_SUBSTR]
PER = divisor for instruction counts (e.g. B*(K+1) -> per instance-iteration)."""
import collections, csv, re, sys

RANGES = [  # (name, first, last) lines of bmc_kernel.cuh
    ("coll", 431, 528), ("cull", 530, 565), ("B.theta", 567, 603),
    ("D2.mma", 628, 659), ("D1.eval", 660, 718), ("D1.cullclk", 719, 746),
    ("D1.collcall", 747, 764), ("D1.U", 765, 791), ("h.assembly", 792, 846),
    ("prologue", 855, 1045), ("A", 1046, 1113), ("C", 1114, 1144), ("D.call", 1145, 1154),
    ("E", 1155, 1173), ("epilogue", 1174, 1252), ("helpers", 161, 430),
]


def frame_phase(chain):
    for f, ln in chain:
        if f.endswith("bmc_kernel.cuh"):
            for name, lo, hi in RANGES:
                if lo <= ln <= hi and name != "helpers":
                    return name
    return "other"


def main():
    dis, src, per = sys.argv[1], sys.argv[2], float(sys.argv[3])
    ksel = sys.argv[4] if len(sys.argv) > 4 else "bmc_am_kernelILi3ELi2E"
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
