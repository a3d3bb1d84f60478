set -u
OUT=gpurun_out/ncudiag2; mkdir -p $OUT
W="python tools/trace_decode.py --ncu --steps 5"
for kb in 0 128 256 512; do
  NFB_PREFETCH_KB=$kb timeout 300 python bench.py --steps 64 --warmup 5 --no-cpu-baseline > $OUT/bench_pf$kb.json 2>&1; echo "pf $kb: $(python -c "import json,sys;d=json.load(open('$OUT/bench_pf$kb.json'));print(d['value'],d['roofline']['frac'])" 2>&1 | tail -1)"
done
NFB_NO_COOP=1 timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:decode_kernel -s 2 -c 3 --csv --log-file $OUT/launches_nocoop.csv $W > $OUT/l1.log 2>&1; echo "nocoop $?"
NFB_NO_COOP=1 NFB_MAX_CLUSTERS=60 timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:decode_kernel -s 2 -c 3 --csv --log-file $OUT/launches_nocoop60.csv $W > $OUT/l2.log 2>&1; echo "nocoop60 $?"
NFB_MAX_CLUSTERS=60 timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:decode_kernel -s 2 -c 3 --csv --log-file $OUT/launches_60.csv $W > $OUT/l3.log 2>&1; echo "coop60 $?"
timeout 100 python tools/trace_decode.py --ncu --steps 5 > $OUT/plain.log 2>&1; echo "plain $?"
ls -la $OUT
