#!/bin/bash
# quick GPU check (dev aid): timings of every config, per-phase profile, GPU tests
# usage: tools/gpu_quick.sh TAG
TAG=${1:-quick}
LOG=gpurun_out/$TAG.log
for c in C3 C4 C2 C1 C5; do timeout -s KILL 120 python tools/timecfg.py $c >> $LOG 2>&1; done
tools/prof_run.sh "C3" "C4" >> $LOG 2>&1
timeout -s KILL 900 python -m pytest tests -m gpu -q -x -p no:cacheprovider > gpurun_out/${TAG}_pytest.log 2>&1
echo pytest rc=$?; tail -3 gpurun_out/${TAG}_pytest.log
