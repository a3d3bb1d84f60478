#!/usr/bin/env bash
# One ncu --set full capture (with source) of one decode launch + per-line
# stall summary.  gpurun -- bash tools/ncu_src.sh TAG
set -u
TAG=${1:-ncu}; OUT=gpurun_out/$TAG; mkdir -p $OUT
NFB_NO_COOP=1 timeout 900 ncu --set full --import-source on --clock-control none -k regex:decode_kernel -s 3 -c 1 \
  -o $OUT/prof -f python tools/trace_decode.py --ncu --steps 4 > $OUT/full.log 2>&1
echo "ncu exit $?"
ncu -i $OUT/prof.ncu-rep --page raw --csv > $OUT/prof_raw.csv 2>/dev/null
ncu -i $OUT/prof.ncu-rep --page source --csv --print-source sass > $OUT/prof_sass.csv 2>/dev/null
ls -la $OUT
