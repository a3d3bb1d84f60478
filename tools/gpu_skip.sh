#!/bin/bash
# Decomposition of the batched step: the same bench with parts of each layer
# skipped (NFB_BATCH_SKIP bits: 1 MLP branch, 2 attention branch, 4 GEMMs).
cd "$(dirname "$0")/.."
OUT=gpurun_out/skip; mkdir -p $OUT
timeout 600 python -m pytest tests/test_split_helpers.py -q -m gpu > $OUT/split_pytest.log 2>&1; echo "split rc=$?" >> $OUT/split_pytest.log
for B in ${BATCHES:-4 16}; do
  for s in 0 1 2 4 5 6 3 7; do
    NFB_BATCH_SKIP=$s timeout 300 python bench.py --batch $B --steps 16 --warmup 3 --no-cpu-baseline > $OUT/b${B}_s$s.json 2> $OUT/b${B}_s$s.err
    python - "$OUT/b${B}_s$s.json" $B $s <<'PY'
import json,sys
try:
    d=json.loads(open(sys.argv[1]).read().strip().splitlines()[-1]); print(f"B={sys.argv[2]} skip={sys.argv[3]} ms/step={d['ms_per_step']:.3f} tok/s={d['value']:.0f} sm={d['clocks']['sm_mhz']}")
except Exception as e: print("fail", sys.argv[2:], e)
PY
  done
done | tee $OUT/summary.txt
