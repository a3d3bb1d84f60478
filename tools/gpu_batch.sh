#!/bin/bash
# Batched path check: GEMM unit tests + batched parity tests, umma microbench, C4 sweep.
cd "$(dirname "$0")/.."
mkdir -p gpurun_out/b
timeout 600 python -m pytest tests/test_gpu_umma.py tests/test_gpu_parity.py -q -m gpu -k "umma or batch or prefill or blocked" > gpurun_out/b/pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/b/pytest.log
timeout 300 python tools/bench_umma.py > gpurun_out/b/umma.jsonl 2>&1
bash tools/bench_batch.sh ${BATCHES:-1 4 16 64} > gpurun_out/b/batch.log 2>&1
tail -3 gpurun_out/b/pytest.log; cat gpurun_out/b/batch.log
python -c "
import json
for l in open('gpurun_out/b/umma.jsonl'):
  try: d=json.loads(l)
  except Exception: print(l.strip()); continue
  print(d['gemm'],d['M'],d['K'],'N',d['N'],'us %.1f'%d['us'],'GB/s %.0f'%d['weight_GBps'])"
