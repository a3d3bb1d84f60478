set -u
OUT=gpurun_out/dbg; mkdir -p $OUT
for m in 0 1 2 3; do
  NFB_DEBUG=$m timeout 300 python bench.py --steps 32 --warmup 3 --no-cpu-baseline > $OUT/bench_d$m.json 2>&1
  echo "debug $m: $(python -c "import json;d=json.load(open('$OUT/bench_d$m.json'));print(round(d['value'],1), round(d['ms_per_step']*1000,1),'us')" 2>&1 | tail -1)"
  NFB_DEBUG=$m timeout 300 python tools/trace_decode.py --out $OUT/trace_d$m.json > $OUT/trace_d$m.log 2>&1
done
