#!/bin/bash
# Interleaved A/B of two builds of the library on the batched bench (clocks
# vary box to box, so both builds run on the same box, alternating):
#   tools/ablib/lib_base.so vs tools/ablib/lib_new.so (git-ignored *.so, they
#   travel with the gpurun snapshot).  BATCHES / REPS override the sweep.
cd "$(dirname "$0")/.."
for rep in $(seq ${REPS:-2}); do for B in ${BATCHES:-4 16 64}; do for L in base new; do
  NFB_LIB=tools/ablib/lib_$L.so timeout 300 python bench.py --batch $B --steps 16 --warmup 3 --no-cpu-baseline 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('B=$B $L', round(d['ms_per_step'],3), round(d['value']), round(d['roofline']['frac'],3), d['clocks']['sm_mhz'])"
done; done; done
