#!/usr/bin/env python
"""Summarise the batched-path ncu evidence (tools/gpu_umma_prof.sh output in
gpurun_out/up/) into one JSON document for profiles/: per captured tcgen05
GEMM launch its duration, DRAM bytes and GB/s, tensor-pipe and TMEM-pipe
activity; the B = 4 bench step's launch list per kernel (cold and warm L2);
and the GEMM microbenchmark lines (no profiler)."""
import collections
import csv
import io
import json
import subprocess
import sys

SRC = sys.argv[1] if len(sys.argv) > 1 else "gpurun_out/up"
OUT = sys.argv[2] if len(sys.argv) > 2 else "profiles/r02_ncu_umma_summary.json"
KEYS = {
    "duration_us": "gpu__time_duration.sum",
    "dram_read_MB": "dram__bytes_read.sum",
    "dram_read_TBps": "dram__bytes_read.sum.per_second",
    "dram_pct_of_peak": "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
    "tensor_pipe_active_pct": "TPC.TriageCompute.sm__pipe_tensor_cycles_active_realtime.avg.pct_of_peak_sustained_elapsed",
    "tc_inst_pct_active": "sm__inst_executed_pipe_tc.avg.pct_of_peak_sustained_active",
    "tmem_inst_pct_active": "sm__inst_executed_pipe_tmem.avg.pct_of_peak_sustained_active",
    "mem_tensor_cycles_pct": "sm__mem_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed",
    "grid": "launch__grid_size",
    "regs": "launch__registers_per_thread",
    "smem_dyn_KB": "launch__shared_mem_per_block_dynamic",
    "sm_clock_GHz": "sm__cycles_elapsed.avg.per_second",
}


def raw(rep):
    txt = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    r = list(csv.reader(io.StringIO(txt)))
    return dict(zip(r[0], r[2])), dict(zip(r[0], r[1]))


def launches(path):
    rows = list(csv.reader(open(path)))
    hi = [i for i, r in enumerate(rows) if "Kernel Name" in r][0]
    h = rows[hi]
    ki, mi, vi, ii = h.index("Kernel Name"), h.index("Metric Name"), h.index("Metric Value"), h.index("ID")
    per = collections.defaultdict(dict)
    for r in rows[hi + 1:]:
        per[int(r[ii])]["k"] = r[ki].split("(")[0]
        per[int(r[ii])][r[mi]] = float(r[vi].replace(",", ""))
    ids = sorted(per)
    start = [i for i in ids if "embed" in per[i]["k"]][-1]  # the last (timed) step
    agg = collections.defaultdict(lambda: [0, 0.0, 0.0])
    for i in ids:
        if i < start:
            continue
        a = agg[per[i]["k"]]
        a[0] += 1
        a[1] += per[i].get("gpu__time_duration.sum", 0)
        a[2] += per[i].get("dram__bytes_read.sum", 0) + per[i].get("dram__bytes_write.sum", 0)
    tot = sum(a[1] for a in agg.values())
    return {"serialised_step_us": round(tot / 1e3, 1), "kernels": {
        k: {"launches": a[0], "us": round(a[1] / 1e3, 1), "share": round(a[1] / tot, 3),
            "dram_MB": round(a[2] / 1e6, 1), "GBps": round(a[2] / max(a[1], 1), 0)}
        for k, a in sorted(agg.items(), key=lambda x: -x[1][1])}}


doc = {"what": "batched path (C4) ncu evidence: tcgen05 GEMM captures (--set full, one launch each, cold, "
               "serialised), the B = 4 bench step's launch list, GEMM microbenchmark without profiler",
       "commands": "tools/gpu_umma_prof.sh", "gemm_captures": {}}
for tag in ("umma_up_16", "umma_qkv_4", "umma_down_64"):
    v, u = raw(f"{SRC}/{tag}.ncu-rep")
    e = {"kernel": v.get("Kernel Name")}
    for k, m in KEYS.items():
        x = v.get(m)
        e[k] = float(x) if x not in (None, "") else None
    doc["gemm_captures"][tag] = e
doc["b4_step_launch_list_cold"] = launches(f"{SRC}/b4_launches.csv")
doc["b4_step_launch_list_warm_l2"] = launches(f"{SRC}/b4_launches_warm.csv")
doc["gemm_microbench"] = [json.loads(x) for x in open(f"{SRC}/umma_bench.jsonl") if x.strip()]
doc["reading"] = ("The projections at N = 2B <= 128 rows are weight-bandwidth bound (arithmetic intensity N "
                  "flop/byte, below the ~340 flop/byte ridge): the tensor pipe is active <1 % of the launch and "
                  "the kernel is a weight stream. Standalone (cold, serialised, three launches per call in the "
                  "microbenchmark) a 40-50 MB projection takes 14-16 us of which ~5 us is launch + first-byte "
                  "latency; inside the step graph the producer's first ring-full of weight copies is issued "
                  "before griddepcontrol.wait (PDL), overlapping the previous kernels.")
json.dump(doc, open(OUT, "w"), indent=1)
print(json.dumps({k: doc["gemm_captures"][k]["duration_us"] for k in doc["gemm_captures"]}))
