#!/bin/bash
# development loop on the GPU box: timings, per-phase profile, cmp vs tools/prev, GPU tests
# usage: tools/iter.sh TAG [notest]
TAG=${1:-it}; LOG=gpurun_out/$TAG.log; mkdir -p gpurun_out
for c in "C3" "C4" "C5" "C2" "C1"; do timeout -s KILL 120 python tools/timecfg.py $c 2>&1 | grep -E "^ C"; done > $LOG
BMC_TEAM=2 timeout -s KILL 120 python tools/timecfg.py C3 148 2>&1 | grep -E "^ C" >> $LOG
cp paper_2109_13030_b200/libbmc.so /tmp/libbmc_keep.so
cp paper_2109_13030_b200/libbmc_prof.so paper_2109_13030_b200/libbmc.so
for a in "C3" "C3 148"; do BMC_TEAM=2 BMC_PROF=1 timeout -s KILL 120 python tools/timecfg.py $a 2>&1 | grep -E "prof" | head -4; done >> $LOG
cp /tmp/libbmc_keep.so paper_2109_13030_b200/libbmc.so
if [ -f tools/prev/libbmc_prev.so ]; then tools/cmp_session.sh ${TAG}_cmp 2>&1 | grep -v bitwise >> $LOG; fi
if [ "$2" != "notest" ]; then
  timeout -s KILL 900 python -m pytest tests -m gpu -q -x -p no:cacheprovider > gpurun_out/${TAG}_pytest.log 2>&1
  echo "pytest rc=$?" >> $LOG; tail -3 gpurun_out/${TAG}_pytest.log >> $LOG
fi
cat $LOG
