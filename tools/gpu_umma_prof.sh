#!/bin/bash
# Batched-path evidence: tcgen05 GEMM microbench (no profiler), ncu --set full
# of one GEMM launch (tensor-pipe + DRAM metrics), the B = 4 bench step's launch
# list, and a full capture of the B = 4 attention tile kernel.
cd "$(dirname "$0")/.."
OUT=gpurun_out/up; mkdir -p $OUT
NCU=/usr/local/cuda/bin/ncu
nvidia-smi --query-gpu=clocks.sm,clocks.max.sm,power.draw --format=csv > $OUT/box.txt
timeout 300 python tools/bench_umma.py > $OUT/umma_bench.jsonl 2> $OUT/umma_bench.err
for sb in up:16 qkv:4 down:64; do
  s=${sb%:*}; b=${sb#*:}
  UMMA_SHAPES=$s UMMA_B=$b UMMA_REPS=2 timeout 300 $NCU --set full --clock-control none --import-source on \
    -k regex:umma_gemm -s 6 -c 1 -o $OUT/umma_${s}_$b python tools/bench_umma.py > $OUT/umma_${s}_$b.txt 2>&1
done
timeout 600 $NCU --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none \
  --csv --log-file $OUT/b4_launches.csv python bench.py --batch 4 --steps 1 --warmup 3 --no-cpu-baseline > $OUT/b4_stdout.txt 2>&1
timeout 600 $NCU --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --cache-control none \
  --csv --log-file $OUT/b4_launches_warm.csv python bench.py --batch 4 --steps 1 --warmup 3 --no-cpu-baseline > $OUT/b4w_stdout.txt 2>&1
timeout 300 $NCU --set full --clock-control none --import-source on -k regex:attn_tile -s 40 -c 1 -o $OUT/attn_b4 \
  python bench.py --batch 4 --steps 1 --warmup 3 --no-cpu-baseline > $OUT/attn_b4.txt 2>&1
ls -la $OUT
