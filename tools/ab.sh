#!/bin/bash
# A/B bench lines: each argument is "ENV=val ENV2=val|extra bench args" (use "-" for defaults).
cd "$(dirname "$0")/.."
mkdir -p gpurun_out/ab
i=0
for spec in "$@"; do
  envs="${spec%%|*}"; args="${spec#*|}"; [ "$args" = "$spec" ] && args=""
  [ "$envs" = "-" ] && envs=""
  env $envs timeout 600 python bench.py --steps ${STEPS:-64} --warmup 5 --no-cpu-baseline $args > gpurun_out/ab/$i.json 2> gpurun_out/ab/$i.err
  echo "[$spec] $(python -c "import json;d=json.load(open('gpurun_out/ab/$i.json'));print(round(d['value'],1),'tok/s',round(d['ms_per_step']*1000,1),'us frac',round(d['roofline']['frac'],3),'e2e',round(d['e2e']['value'],1), d['config'].get('autotune'), d['clocks']['sm_mhz'])" 2>&1 | tail -1)"
  i=$((i+1))
done
