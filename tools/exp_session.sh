#!/bin/bash
# Experiment session (dev aid): A/B timings of library variants + PROFILE-build phase cycles.
#   LIBS="libbmc.so libbmc_x.so" PROFS="libbmc_prof.so libbmc_xprof.so" CFGS="C3 C4 C5" tools/exp_session.sh TAG
TAG=${1:-exp}; LOG=gpurun_out/$TAG.log; mkdir -p gpurun_out; : > $LOG
for rep in 1 2; do
  for lib in ${LIBS:-libbmc.so}; do
    for c in ${CFGS:-C3 C4}; do
      BMC_LIB=paper_2109_13030_b200/$lib timeout -s KILL 120 python tools/timecfg.py $c 2>&1 | grep -E "^ C|^paper|rror" >> $LOG
    done
  done
done
for lib in ${PROFS:-}; do
  for c in ${PCFGS:-C3}; do
    echo "== PROFILE $lib $c" >> $LOG
    BMC_PROF=1 BMC_LIB=paper_2109_13030_b200/$lib timeout -s KILL 120 python tools/timecfg.py $c 2>&1 | grep -E "prof\]" | tail -6 >> $LOG
  done
done
if [ -n "$EXTRA" ]; then bash -c "$EXTRA" >> $LOG 2>&1; fi
cat $LOG
