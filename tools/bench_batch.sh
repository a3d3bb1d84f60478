#!/usr/bin/env bash
# BASELINE configs[3]: Pythia-2.8B batch sweep at context 4096.
set -u
OUT=gpurun_out/batch; mkdir -p $OUT
for B in "$@"; do
  timeout 900 python bench.py --batch $B --steps 16 --warmup 3 --no-cpu-baseline > $OUT/b_$B.json 2> $OUT/b_$B.err
  echo "B=$B $(python -c "import json;d=json.load(open('$OUT/b_$B.json'));print(round(d['value'],1),'tok/s', round(d['ms_per_step'],3),'ms/step frac', round(d['roofline']['frac'],3), 'e2e', round(d['e2e']['value'],1))" 2>&1 | tail -1)"
done
