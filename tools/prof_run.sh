#!/bin/bash
# per-phase cycle profile with the PROFILE=1 library (dev aid)
cp paper_2109_13030_b200/libbmc.so /tmp/libbmc_keep.so
cp paper_2109_13030_b200/libbmc_prof.so paper_2109_13030_b200/libbmc.so
for args in "$@"; do BMC_PROF=1 timeout -s KILL 120 python tools/timecfg.py $args 2>&1 | grep -E "prof|^C" | head -8; done
cp /tmp/libbmc_keep.so paper_2109_13030_b200/libbmc.so
