#!/usr/bin/env bash
# Bench + trace under several env settings.  Each argument is one setting,
# e.g. "NFB_CLUSTER=4 NFB_HEAD_WEIGHT=150".
#   gpurun -- bash tools/sweep.sh TAG "SETTING" ...
set -u
TAG=$1; shift
OUT=gpurun_out/$TAG; mkdir -p $OUT
i=0
for cfg in "$@"; do
  i=$((i+1))
  env $cfg timeout 300 python bench.py --steps 64 --warmup 5 --no-cpu-baseline > $OUT/bench_$i.json 2> $OUT/bench_$i.err
  r=$(python -c "import json;d=json.load(open('$OUT/bench_$i.json'));print(round(d['value'],1), round(d['ms_per_step']*1000,1),'us frac', round(d['value']*5650524160/6.55e12,3), d['clocks']['sm_mhz'])" 2>&1 | tail -1)
  env $cfg timeout 120 python tools/trace_decode.py --out $OUT/trace_$i.json > $OUT/trace_$i.log 2>&1
  t=$(python -c "
import json;d=json.load(open('$OUT/trace_$i.json'));s=d['summary']
print('layer',round(s['layer_us'],2),'work',round(s['work_us_med'],1),round(s['work_us_max'],1),'head',round(s['work_us_head_med'],1),'mlp',round(s['work_us_mlp_med'],1),'bar1w',round(s['bar1_wait_us_med'],2),'red',round(s['cluster_reduce_us_med'],2),'fold+b2',round(s['fold_bar2_us_med'],2),'hd',round(d['head_phase_us'],1))" 2>&1 | tail -1)
  echo "[$cfg] $r | $t"
done
