#!/bin/bash
# ncu summary of a round session's C3 capture with the per-phase attribution (dev aid):
#   tools/ncu_report.sh VER   (reads gpurun_out/r2_VER/prof.ncu-rep, writes profiles/r2_c3_VER.md)
# The disassembly comes from the in-tree libbmc.so, which must be the captured build.
set -e
V=$1; REP=gpurun_out/r2_$V/prof.ncu-rep; TMP=$(mktemp -d)
KSEL=${KSEL:-bmc_am_kernelILi3ELi2ELb0ELb1ELb1E}   # the C3 launch (circles: ELLK false)
python tools/ncu_summary.py $REP r2_c3_$V > /dev/null
(cd $TMP && cuobjdump -xelf all /root/repo/paper_2109_13030_b200/libbmc.so > /dev/null)
CUBIN=$(grep -l "$KSEL" $TMP/*.cubin | head -1)
nvdisasm -gi $CUBIN > $TMP/dis.txt
ncu -i $REP --page source --csv --print-source sass > $TMP/src.csv
{ echo; echo "## Per-phase attribution (tools/ncu_phases.py, per instance-iteration; B = 1000 x 101 evaluations)"; echo
  echo '```'; python tools/ncu_phases.py $TMP/dis.txt $TMP/src.csv 101000 $KSEL; echo '```'; } >> profiles/r2_c3_$V.md
rm -rf $TMP
