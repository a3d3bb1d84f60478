# quick GPU check: parity tests + bench + trace (+ optional debug modes)
set -u
TAG=${1:-q}; OUT=gpurun_out/$TAG; mkdir -p $OUT
[ -n "${NO_TEST:-}" ] || timeout 600 python -m pytest tests -x -q -m gpu > $OUT/pytest.log 2>&1; echo "pytest: $(tail -1 $OUT/pytest.log)"
timeout 300 python bench.py --steps 64 --warmup 5 --no-cpu-baseline > $OUT/bench.json 2> $OUT/bench.err
echo "bench: $(python -c "import json;d=json.load(open('$OUT/bench.json'));print(round(d['value'],1), round(d['ms_per_step']*1000,1),'us', round(d['roofline']['frac'],3), d['clocks'])" 2>&1 | tail -1)"
timeout 120 python tools/trace_decode.py --out $OUT/trace.json > $OUT/trace.log 2>&1
python -c "
import json;d=json.load(open('$OUT/trace.json'));s=d['summary']
print('trace kernel',round(d['kernel_us']),'pw',round(d['producer_wait_us_med']),'cw',round(d['consumer_wait_us_med']),'head',round(d['head_phase_us']), {k:round(v,2) for k,v in s.items() if k in ('work_us_med','work_us_head_med','work_us_mlp_med','qkv_us_head_med','ctx_us_head_med','cluster_reduce_us_med','bar1_us_med','fold_us_med','bar2_us_med','layer_us')})"
for m in ${DBG:-}; do
  NFB_DEBUG=$m timeout 120 python bench.py --steps 32 --warmup 3 --no-cpu-baseline > $OUT/bench_d$m.json 2>&1
  echo "debug $m: $(python -c "import json;d=json.load(open('$OUT/bench_d$m.json'));print(round(d['value'],1), round(d['ms_per_step']*1000,1),'us')" 2>&1 | tail -1)"
done
