#!/bin/bash
# Round-2 evidence pass: ncu launch list of the bench command itself, and
# compute-sanitizer passes over the sanitize workload.
cd "$(dirname "$0")/.."
OUT=gpurun_out/prof2; mkdir -p $OUT
NCU=/usr/local/cuda/bin/ncu
NFB_AUTOTUNE=0 timeout 900 $NCU --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -c 600 --csv --log-file $OUT/bench_launches.csv python bench.py --steps 4 --warmup 3 --no-cpu-baseline > $OUT/bench_under_ncu.txt 2>&1
echo "ncu rc=$?"
bash tools/sanitize.sh
