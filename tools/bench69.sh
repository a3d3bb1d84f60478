#!/usr/bin/env bash
# Pythia-6.9B (BASELINE configs[2]) bench lines under a few settings.
set -u
OUT=gpurun_out/b69; mkdir -p $OUT
i=0
for cfg in "$@"; do
  i=$((i+1))
  env $cfg timeout 600 python bench.py --model pythia-6.9b --steps 32 --warmup 3 --no-cpu-baseline > $OUT/b_$i.json 2> $OUT/b_$i.err
  echo "[$cfg] $(python -c "import json;d=json.load(open('$OUT/b_$i.json'));print(round(d['value'],1), round(d['ms_per_step']*1000,1),'us frac', round(d['roofline']['frac'],3))" 2>&1 | tail -1)"
done
