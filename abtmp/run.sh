cd /root/repo
for rep in 1 2; do for B in 4 16 64; do for L in base new; do
NFB_LIB=abtmp/lib_$L.so timeout 300 python bench.py --batch $B --steps 16 --warmup 3 --no-cpu-baseline 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('B=$B $L', round(d['ms_per_step'],3), round(d['value']), round(d['roofline']['frac'],3), d['clocks']['sm_mhz'])"
done; done; done
