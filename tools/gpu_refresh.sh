#!/bin/bash
# Evidence refresh of the final code: full GPU suite (parity report), smoke,
# C2 headline bench, C3 bench line, C4 batch sweep.
cd "$(dirname "$0")/.."
O=gpurun_out/refresh; mkdir -p $O
nvidia-smi --query-gpu=name,clocks.max.sm,power.limit --format=csv > $O/box.txt
python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo "smoke rc=$?" >> $O/smoke.log
rm -f $O/parity.jsonl
NFB_PARITY_REPORT=$O/parity.jsonl timeout 1500 python -m pytest tests -m gpu -q -rA -p no:cacheprovider > $O/pytest.log 2>&1; echo "pytest rc=$?" >> $O/pytest.log
timeout 600 python bench.py --steps 128 --warmup 5 > $O/bench.json 2> $O/bench.err
timeout 900 python bench.py --model pythia-6.9b --steps 64 --warmup 5 > $O/bench_c3.json 2> $O/bench_c3.err
for B in 1 4 16 64; do
  timeout 600 python bench.py --batch $B --steps 16 --warmup 3 --no-cpu-baseline > $O/batch_$B.json 2> $O/batch_$B.err
done
tail -2 $O/pytest.log; tail -1 $O/smoke.log
for f in bench bench_c3 batch_1 batch_4 batch_16 batch_64; do python -c "
import json; d=json.loads(open('$O/$f.json').read().strip().splitlines()[-1]); print('$f', round(d['value'],1), round(d['roofline']['frac'],3), d.get('e2e',{}).get('value'), d['clocks'])" 2>&1 | tail -1; done
