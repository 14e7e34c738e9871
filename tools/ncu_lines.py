"""Development aid: attribute ncu per-SASS metrics (source page, --print-source sass)
to CUDA source lines via an `nvdisasm -g` listing of the same cubin.

usage: python tools/ncu_lines.py DIS.txt SRC.csv KERNEL.cuh [top] [per]
  DIS.txt  : nvdisasm -g (or -gi with OUTER=1: attribute inlined code to its call site) -c <cubin extracted with cuobjdump -xelf all>
  SRC.csv  : ncu -i rep --page source --csv --print-source sass
  per      : divisor for instruction counts (e.g. B*(K+1) -> per instance-iteration)
Prints the heaviest lines by executed warp instructions and a per-range summary
when RANGES (name:first-last,...) is set in the environment."""
import collections
import csv
import os
import re
import sys

OUTER = os.environ.get('OUTER') == '1'


def load(dis_path, csv_path):
    dis = open(dis_path).read().split('\n')
    insts, in_k, cur = [], False, ('?', 0)
    for l in dis:
        if l.strip().startswith('.section') and '.text.' in l:
            in_k = os.environ.get('KSEL', 'bmc_am_kernel') in l
            continue
        if not in_k:
            continue
        m = re.search(r'//## File "([^"]+)", line (\d+)(.*)', l)
        if m:
            cur = (m.group(1).split('/')[-1], int(m.group(2)))
            if OUTER:   # attribute to the outermost frame (needs an nvdisasm -gi listing)
                chain = [cur] + [(a.split('/')[-1], int(b)) for a, b in
                                 re.findall(r'inlined at "([^"]+)", line (\d+)', m.group(3))]
                cur = chain[-1]
            continue
        m = re.match(r'\s*/\*([0-9a-f]{4,})\*/\s+(.*)', l)
        if m:
            insts.append((cur[0], cur[1], m.group(2).split(';')[0].strip()))
    rows = list(csv.reader(open(csv_path)))
    idx = {h: i for i, h in enumerate(rows[1])}
    data = rows[2:]
    base = int(data[0][0], 16)
    n_by, s_by = collections.Counter(), collections.Counter()
    for r in data:
        k = (int(r[0], 16) - base) // 16
        key = f"{insts[k][0]}:{insts[k][1]}" if k < len(insts) else '?'
        n_by[key] += float(r[idx['Instructions Executed']] or 0)
        s_by[key] += float(r[idx['Warp Stall Sampling (All Samples)']] or 0)
    return n_by, s_by


def main():
    dis_path, csv_path, src_path = sys.argv[1:4]
    top = int(sys.argv[4]) if len(sys.argv) > 4 else 40
    per = float(sys.argv[5]) if len(sys.argv) > 5 else 1.0
    n_by, s_by = load(dis_path, csv_path)
    src = open(src_path).read().split('\n')
    base = os.path.basename(src_path)
    tn, ts = sum(n_by.values()), sum(s_by.values()) or 1.0
    print(f"total inst {tn / per:.1f}")
    for key, n in n_by.most_common(top):
        f, ln = key.split(':') if ':' in key else ('?', '0')
        text = src[int(ln) - 1].strip()[:78] if f == base else ''
        print(f"{key:26s} inst {n / per:8.1f} stall {100 * s_by[key] / ts:5.1f}% {text}")
    if os.environ.get('RANGES'):
        for item in os.environ['RANGES'].split(','):
            name, rg = item.split(':')
            lo, hi = map(int, rg.split('-'))
            n = sum(v for k, v in n_by.items() if k.startswith(base + ':') and lo <= int(k.split(':')[1]) <= hi)
            s = sum(v for k, v in s_by.items() if k.startswith(base + ':') and lo <= int(k.split(':')[1]) <= hi)
            print(f"range {name:10s} inst {n / per:8.1f} stall {100 * s / ts:5.1f}%")


if __name__ == '__main__':
    main()
