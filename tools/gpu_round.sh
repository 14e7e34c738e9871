#!/bin/bash
# Round-level GPU session (dev aid): GPU tests, bench lines, ncu launch list + full
# capture of the C3 launch, sweeps and the required-work count.
# usage: tools/gpu_round.sh TAG
TAG=${1:-round}; OUT=gpurun_out/$TAG; mkdir -p $OUT
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv > $OUT/nvsmi.txt
timeout 2400 python -m pytest tests -m gpu -q -p no:cacheprovider -s > $OUT/pytest_gpu.log 2>&1; echo "pytest rc=$?"
tail -3 $OUT/pytest_gpu.log
timeout 600 python bench.py --steps 20 --warmup 5 > $OUT/bench.log 2>&1; echo "bench rc=$?"
timeout 600 python bench.py --steps 10 --warmup 3 --strong 16384 --no-cpu-baseline > $OUT/bench_strong.log 2>&1; echo "strong rc=$?"
timeout 600 python bench.py --steps 10 --warmup 3 --ellipse 1 --no-cpu-baseline > $OUT/bench_ell1.log 2>&1; echo "ell rc=$?"
timeout 600 python bench.py --steps 10 --warmup 3 --config C4 --no-cpu-baseline > $OUT/bench_c4.log 2>&1; echo "c4 rc=$?"
CMD="python bench.py --steps 1 --warmup 3 --no-cpu-baseline"
timeout 300 $CMD > $OUT/plain.log 2>&1 && \
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $OUT/launches.csv $CMD > $OUT/ncu_launch.log 2>&1; echo "ncu-launch rc=$?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:bmc_am_kernel -s 3 -c 1 -o $OUT/prof $CMD > $OUT/ncu_full.log 2>&1; echo "ncu-full rc=$?"
timeout 900 python tools/sweeps.py $OUT/sweeps.json > $OUT/sweeps.md 2>&1; echo "sweeps rc=$?"
timeout 300 python tools/required_work.py C3 C4 > $OUT/required_work.log 2>&1; echo "required rc=$?"
cp profiles/required_work.json $OUT/ 2>/dev/null
tail -2 $OUT/bench.log
