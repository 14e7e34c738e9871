#!/bin/bash
# Quick A/B timing of library variants on chosen configs (development aid):
#   CFGS="C3 C4" tools/abq.sh TAG lib1 lib2 ...
TAG=$1; shift; LOG=gpurun_out/$TAG.log; mkdir -p gpurun_out; : > $LOG
for rep in 1 2; do
for lib in "$@"; do
  for c in ${CFGS:-C3 C4}; do BMC_LIB=paper_2109_13030_b200/$lib timeout -s KILL 120 python tools/timecfg.py $c 2>&1 | grep -E "^ C|^paper|rror" ; done >> $LOG
done; done
cat $LOG
