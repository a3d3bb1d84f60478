#!/usr/bin/env python
"""Summarise an `ncu --set full` raw CSV (ncu -i X.ncu-rep --page raw --csv) and
an ncu launch list (--metrics gpu__time_duration.sum --csv) into the JSON kept
under profiles/.

    python tools/ncu_summary.py RAW.csv LAUNCHES.csv OUT.json [--bytes B]
"""
import csv
import json
import sys

KEYS = [
    "gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
    "dram__bytes.sum.per_second", "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
    "sm__throughput.avg.pct_of_peak_sustained_elapsed", "sm__cycles_elapsed.avg.per_second",
    "launch__registers_per_thread", "launch__grid_size", "launch__block_size",
    "launch__cluster_dim_x", "launch__shared_mem_per_block_dynamic", "smsp__inst_executed.sum",
    "lts__t_sector_hit_rate.pct", "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum",
    "smsp__warps_active.avg.pct_of_peak_sustained_active",
]
SCALE = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "Tbyte": 1e12,
         "ns": 1e-9, "us": 1e-6, "usecond": 1e-6, "ms": 1e-3, "msecond": 1e-3, "s": 1.0}


def num(v, unit):
    v = float(v.replace(",", ""))
    base = unit.split("/")[0]
    return v * SCALE.get(base, 1.0)


def main():
    raw, launches, out = sys.argv[1:4]
    algo = None
    if "--bytes" in sys.argv:
        algo = float(sys.argv[sys.argv.index("--bytes") + 1])
    rows = list(csv.reader(open(raw)))
    hdr, units = rows[0], rows[1]
    res = {"kernel": None, "metrics": {}}
    for r in rows[2:]:
        d = dict(zip(hdr, r))
        res["kernel"] = d.get("Kernel Name")
        for k in KEYS:
            if k in d:
                res["metrics"][k] = {"value": d[k], "unit": units[hdr.index(k)]}
        break
    m = res["metrics"]
    rd = num(m["dram__bytes_read.sum"]["value"], m["dram__bytes_read.sum"]["unit"])
    wr = num(m["dram__bytes_write.sum"]["value"], m["dram__bytes_write.sum"]["unit"])
    res["dram_bytes_per_launch"] = rd + wr
    if algo:
        res["algorithmic_bytes_per_launch"] = algo
        res["traffic_over_algorithmic"] = (rd + wr) / algo
    lt = []
    lines = [ln for ln in open(launches) if ln.startswith('"')]
    for r in csv.DictReader(lines):
        if r.get("Metric Name") == "gpu__time_duration.sum":
            lt.append(float(r["Metric Value"].replace(",", "")) * SCALE.get(r["Metric Unit"], 1e-9))
    res["launch_list"] = {"n": len(lt), "kernel_s": lt,
                          "mean_s": sum(lt) / len(lt) if lt else None}
    json.dump(res, open(out, "w"), indent=1)
    print(json.dumps({k: v for k, v in res.items() if k != "metrics"}, indent=1))


if __name__ == "__main__":
    main()
