#!/bin/bash
# compute-sanitizer passes over tools/sanitize_workload.py; logs -> gpurun_out/sanitize/.
cd "$(dirname "$0")/.."
OUT=gpurun_out/sanitize; mkdir -p $OUT
CS=/usr/local/cuda/bin/compute-sanitizer
for tool in memcheck synccheck racecheck initcheck; do
  extra=""
  [ $tool = memcheck ] && extra="--leak-check full"
  timeout 900 $CS --tool $tool $extra --print-limit 50 --error-exitcode 3 python tools/sanitize_workload.py > $OUT/$tool.log 2>&1
  echo "$tool rc=$?" | tee -a $OUT/$tool.log
done
