#!/bin/bash
# ncu of the batched path: umma kernel times from the microbench, one B=16 step launch list, one full capture.
cd "$(dirname "$0")/.."
OUT=gpurun_out/nb; mkdir -p $OUT
NCU=/usr/local/cuda/bin/ncu
timeout 600 $NCU --metrics gpu__time_duration.sum,dram__bytes_read.sum --clock-control none -k regex:umma_gemm --csv --log-file $OUT/umma_launches.csv python tools/bench_umma.py > $OUT/umma_ncu_stdout.txt 2>&1
timeout 600 $NCU --metrics gpu__time_duration.sum,dram__bytes_read.sum --clock-control none --csv --log-file $OUT/b16_launches.csv python bench.py --batch ${B:-16} --steps 1 --warmup 3 --no-cpu-baseline > $OUT/b16_stdout.txt 2>&1
timeout 600 $NCU --set full --clock-control none --import-source on -k regex:umma_gemm -s 20 -c 1 -o $OUT/umma_full python tools/bench_umma.py > $OUT/umma_full_stdout.txt 2>&1
ls -la $OUT
