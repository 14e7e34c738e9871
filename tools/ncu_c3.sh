#!/bin/bash
# one ncu --set full capture of the C3 bench launch (dev aid): tools/ncu_c3.sh TAG
TAG=${1:-ncu}; OUT=gpurun_out/$TAG; mkdir -p $OUT
CMD="python bench.py --steps 1 --warmup 3 --no-cpu-baseline"
timeout 300 $CMD > $OUT/plain.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:bmc_am_kernel -s 3 -c 1 -o $OUT/prof $CMD > $OUT/ncu_full.log 2>&1; echo "ncu-full rc=$?"
