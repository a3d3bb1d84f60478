#!/bin/bash
# Final evidence pass: smoke, full GPU suite (parity report), headline bench,
# ncu full capture + source page of the decode kernel, ncu launch list of the
# bench command, reference arm.
cd "$(dirname "$0")/.."
O=gpurun_out/final; mkdir -p $O
python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo "smoke rc=$?" >> $O/smoke.log
rm -f $O/parity.jsonl
NFB_PARITY_REPORT=$O/parity.jsonl timeout 1500 python -m pytest tests -m gpu -q -rA -p no:cacheprovider > $O/pytest.log 2>&1; echo "pytest rc=$?" >> $O/pytest.log
timeout 600 python bench.py --steps 128 --warmup 5 > $O/bench.json 2> $O/bench.err
NCU=/usr/local/cuda/bin/ncu
NFB_NO_COOP=1 timeout 900 $NCU --set full --import-source on --clock-control none -k regex:decode_kernel -s 3 -c 1 -o $O/decode_full -f python tools/trace_decode.py --ncu --steps 4 > $O/ncu_full.log 2>&1
$NCU -i $O/decode_full.ncu-rep --page raw --csv > $O/decode_raw.csv 2>/dev/null
$NCU -i $O/decode_full.ncu-rep --page source --csv --print-source sass > $O/decode_sass.csv 2>/dev/null
NFB_AUTOTUNE=0 timeout 900 $NCU --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -c 600 --csv --log-file $O/bench_launches.csv python bench.py --steps 4 --warmup 3 --no-cpu-baseline > $O/bench_under_ncu.txt 2>&1
timeout 600 python bench.py --impl reference > $O/bench_ref.json 2> $O/bench_ref.err
tail -2 $O/pytest.log; tail -1 $O/smoke.log; head -c 400 $O/bench.json
