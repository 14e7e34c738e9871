#!/bin/bash
# Copy one round session's artifacts (tools/gpu_round.sh) into profiles/ under the
# version tag and summarise the ncu capture (dev aid): tools/collect_round.sh VER
set -e
V=$1; O=gpurun_out/r2_$V
for p in "bench.log r2_c3_${V}_bench.json" "bench_c4.log r2_c4_${V}_bench.json" \
         "bench_strong.log r2_c5_strong16384_${V}_bench.json" "bench_ell1.log r2_c3_ellipses_rule1_${V}_bench.json"; do
  set -- $p; grep '^{' $O/$1 | tail -1 | python -m json.tool > profiles/$2
done
cp $O/launches.csv profiles/r2_c3_${V}_launches.csv
cp $O/sweeps.md profiles/r2_sweeps_${V}.md; cp $O/sweeps.json profiles/r2_sweeps_${V}.json
bash tools/ncu_report.sh $V
python - "$V" <<'PY'
import json, re, sys
v = sys.argv[1]; md = open(f"profiles/r2_c3_{v}.md").read()
get = lambda k: float(re.search(r"\| %s \| ([0-9.]+) \|" % re.escape(k), md).group(1))
rd, wr = get("dram__bytes_read.sum"), get("dram__bytes_write.sum")
issue = get("smsp__issue_active.avg.pct_of_peak_sustained_active")
p = "profiles/dram_traffic.json"; d = json.load(open(p))
d.update(C3_bytes_per_launch=(rd + wr) * 1e3, read=rd * 1e3, write=wr * 1e3, C3_issue_active_pct=round(issue, 1),
         source=f"ncu --set full --clock-control none, one bmc_am_kernel<3,2,false,true,true> launch of bench.py C3 "
                f"(round 2, profiles/r2_c3_{v}.md), dram__bytes_read.sum + dram__bytes_write.sum; "
                "smsp__issue_active.avg.pct_of_peak_sustained_active")
json.dump(d, open(p, "w"), indent=1); open(p, "a").write("\n")
print("traffic", d["C3_bytes_per_launch"], "issue", d["C3_issue_active_pct"])
PY
