#!/bin/bash
# Round-2 GPU pass: smoke, the whole -m gpu suite (parity report), the bench line.
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
( nproc; free -g; nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv ) > gpurun_out/box.txt 2>&1
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/smoke.log
rm -f gpurun_out/parity.jsonl
NFB_PARITY_REPORT=gpurun_out/parity.jsonl timeout 1500 python -m pytest tests -m gpu -q -rA --durations=15 ${PYTEST_ARGS} > gpurun_out/pytest.log 2>&1
echo "pytest rc=$?" >> gpurun_out/pytest.log
if [ -z "$NO_BENCH" ]; then
  timeout 600 python bench.py --steps 128 --warmup 5 > gpurun_out/bench.json 2> gpurun_out/bench.err
  echo "bench rc=$?" >> gpurun_out/bench.err
fi
tail -3 gpurun_out/pytest.log; cat gpurun_out/bench.json 2>/dev/null | head -c 600
