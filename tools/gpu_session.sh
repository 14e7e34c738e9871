#!/bin/bash
# One gpurun session: probe, GPU tests, bench, launch list + one ncu capture.
# usage: tools/gpu_session.sh TAG [skip-tests] [skip-ncu]
TAG=${1:-dev}
OUT=gpurun_out/$TAG
mkdir -p $OUT
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv > $OUT/nvsmi.txt
timeout 300 python tools/probe.py > $OUT/probe.log 2>&1; echo "probe rc=$?"
if [ "$2" != "skip-tests" ]; then
  timeout 900 python -m pytest tests -m gpu -q -p no:cacheprovider -x > $OUT/pytest_gpu.log 2>&1; echo "pytest rc=$?"
fi
timeout 600 python bench.py --steps 10 --warmup 3 > $OUT/bench.log 2>&1; echo "bench rc=$?"
if [ "$3" != "skip-ncu" ]; then
  CMD="python bench.py --steps 1 --warmup 3 --no-cpu-baseline"
  timeout 300 $CMD > $OUT/plain.log 2>&1 && \
  timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $OUT/launches.csv $CMD > $OUT/ncu_launch.log 2>&1; echo "ncu-launch rc=$?"
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:bmc_am_kernel -s 3 -c 1 -o $OUT/prof $CMD > $OUT/ncu_full.log 2>&1; echo "ncu-full rc=$?"
fi
tail -5 $OUT/probe.log; tail -5 $OUT/pytest_gpu.log; cat $OUT/bench.log | tail -3
