#!/usr/bin/env python
"""Close the reference's calibration loop on B200 measurements.

Feeds a measured TPOT CSV (`tools/tpot_csv.py`, the reference's
`seq_len,tpot_ms,variant` format, nf/perfmodel.py:337-398) to the reference's
own `calibrate` (nf/perfmodel.py:455-535) with the bandwidth pinned to the
measured B200 HBM copy bandwidth (MEASURED_PEAKS.json `hbm_gbs`) instead of
the reference's 1.8e12 RTX-5090 default: `calibrate` never fits the
bandwidth, so with the default it has to explain a 4x faster GPU with
efficiencies clamped to <= 1 and the fit degenerates (round 1: max rel error
1.58).  Writes one JSON document (fitted parameters + per-row errors).

Runs only in the build container: it imports the reference from
/root/reference (read-only, never on the GPU box, never in the product).

    python tools/calibrate_b200.py --csv profiles/r02_tpot_pythia28b_b200.csv \
        --out profiles/r02_reference_calibrate_b200.json
"""
import argparse
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
REF = "/root/reference/pkg/src"


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--csv", required=True)
    ap.add_argument("--out", required=True)
    ap.add_argument("--bandwidth", type=float, default=0.0, help="B/s (default: MEASURED_PEAKS.json hbm_gbs)")
    a = ap.parse_args()
    sys.path.insert(0, REF)
    from neoxfuse.config import preset
    from neoxfuse.perfmodel import KERNEL_CLASSES, calibrate, read_measurements_csv

    bw = a.bandwidth
    src = "--bandwidth"
    if bw <= 0:
        peaks = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))
        bw = peaks["hbm_gbs"] * 1e9
        src = "MEASURED_PEAKS.json hbm_gbs"
    ms = read_measurements_csv(a.csv)
    res = calibrate(ms, preset("pythia-2.8b"), bandwidth=bw)
    hw = res.hardware
    doc = {
        "what": "reference calibrate (nf/perfmodel.py:455-535) on measured B200 TPOT",
        "measurements": os.path.relpath(os.path.abspath(a.csv), ROOT),
        "bandwidth_Bps": bw,
        "bandwidth_source": src,
        "free_params": res.free_params,
        "fitted": {
            "efficiency": {c: hw.efficiency[c] for c in KERNEL_CLASSES},
            "launch_overhead_s": hw.launch_overhead,
            "descriptor_cost_s": hw.descriptor_cost,
            "graph_replay_overhead_s": hw.graph_replay_overhead,
        },
        "max_rel_error": res.max_rel_error,
        "rows": [
            {"variant": r.variant, "seq_len": r.seq_len, "measured_ms": r.measured_ms,
             "predicted_ms": r.predicted_ms, "rel_error": r.rel_error}
            for r in res.rows
        ],
    }
    with open(a.out, "w") as f:
        json.dump(doc, f, indent=1)
    print(json.dumps({k: doc[k] for k in ("bandwidth_Bps", "fitted", "max_rel_error")}))


if __name__ == "__main__":
    main()
