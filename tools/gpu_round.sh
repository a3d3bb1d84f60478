#!/usr/bin/env bash
# One gpurun call: GPU parity tests, smoke, bench line, ncu launch list and one
# full ncu capture of the decode kernel.  Outputs land in gpurun_out/.
#   gpurun --timeout 1500 -- bash tools/gpu_round.sh [tag] [parts...]
# parts: tests smoke bench launches benchlaunches full trace (default: all)
set -u
TAG=${1:-r01}
shift || true
PARTS=${*:-"tests smoke bench launches benchlaunches full trace"}
OUT=gpurun_out/$TAG
mkdir -p "$OUT"
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,memory.total --format=csv > "$OUT/gpu.txt" 2>&1
has() { [[ " $PARTS " == *" $1 "* ]]; }
if has tests; then
  timeout 900 python -m pytest tests -x -q -m gpu > "$OUT/pytest_gpu.log" 2>&1
  echo "pytest exit $?" >> "$OUT/pytest_gpu.log"
  tail -3 "$OUT/pytest_gpu.log"
fi
if has smoke; then
  timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > "$OUT/smoke.log" 2>&1
  echo "smoke exit $?" >> "$OUT/smoke.log"
  tail -2 "$OUT/smoke.log"
fi
if has bench; then
  timeout 600 python bench.py > "$OUT/bench.json" 2> "$OUT/bench.err"
  echo "bench exit $?"; tail -c 1500 "$OUT/bench.json"
fi
if has trace; then
  timeout 300 python tools/trace_decode.py --out "$OUT/trace.json" > "$OUT/trace.log" 2>&1
  echo "trace exit $?"
fi
if has launches; then
  NFB_NO_COOP=1 timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:decode_kernel -s 3 -c 6 --csv \
    --log-file "$OUT/launches.csv" python tools/trace_decode.py --ncu --steps 9 > "$OUT/launches.log" 2>&1
  echo "launches exit $?"
fi
if has benchlaunches; then
  # the launch list of the bench command itself (timed region = last 8 launches)
  NFB_AUTOTUNE=0 timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv \
    --log-file "$OUT/bench_launches.csv" python bench.py --steps 8 --warmup 3 --no-cpu-baseline \
    > "$OUT/bench_launches.log" 2>&1
  echo "benchlaunches exit $?"
fi
if has full; then
  NFB_NO_COOP=1 timeout 900 ncu --set full --clock-control none --import-source on -k regex:decode_kernel -s 3 -c 1 \
    -o "$OUT/prof" -f python tools/trace_decode.py --ncu --steps 4 > "$OUT/full.log" 2>&1
  echo "full exit $?"
  ncu -i "$OUT/prof.ncu-rep" --page raw --csv > "$OUT/prof_raw.csv" 2>/dev/null
fi
ls -la "$OUT"
