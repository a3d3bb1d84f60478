#!/bin/bash
# Exploration pass: decode bounds (trace variant no-copy / no-compute), C4 batch sweep, umma microbench.
cd "$(dirname "$0")/.."
mkdir -p gpurun_out/x
NO_TEST=1 DBG="1 2" bash tools/quick.sh x_base > gpurun_out/x/quick.log 2>&1 || true
NFB_DEBUG=1 timeout 120 python tools/trace_decode.py --out gpurun_out/x/trace_nocopy.json > /dev/null 2>&1
NFB_DEBUG=2 timeout 120 python tools/trace_decode.py --out gpurun_out/x/trace_nocompute.json > /dev/null 2>&1
timeout 300 python tools/bench_umma.py > gpurun_out/x/umma.jsonl 2>&1
bash tools/bench_batch.sh 1 4 16 64 > gpurun_out/x/batch.log 2>&1
cat gpurun_out/x/quick.log gpurun_out/x/batch.log
