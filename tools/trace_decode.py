#!/usr/bin/env python
"""Per-CTA phase timeline of one Pythia decode step (device globaltimer stamps).

    python tools/trace_decode.py [--preset pythia-2.8b] [--ctx 1024] [--out gpurun_out/trace.json]

Also usable as the short workload for ncu:  --ncu runs warm-up + N eager steps
without tracing.
"""

import argparse
import json
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from paper_2604_23553_b200 import Engine, mean_step_bytes, preset  # noqa: E402


CYC = 1965.0  # SM clock64 ticks per us (accumulated waits are in cycles)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--preset", default="pythia-2.8b")
    ap.add_argument("--ctx", type=int, default=1024)
    ap.add_argument("--steps", type=int, default=3)
    ap.add_argument("--cluster", type=int, default=0)
    ap.add_argument("--dynamic", action="store_true")
    ap.add_argument("--ncu", action="store_true", help="no tracing; eager steps for a profiler")
    ap.add_argument("--out", default=os.path.join(ROOT, "gpurun_out", "trace.json"))
    a = ap.parse_args()
    cfg = preset(a.preset)
    eng = Engine(cfg, max_seq=a.ctx + a.steps + 8, cluster_size=a.cluster)
    eng.synth_model(0)
    eng.kv_synth_all(a.ctx, 7)
    if a.dynamic:
        eng.set_option("dynamic_mlp", True)
    if not a.ncu:
        eng.set_option("trace", True)
    eng.begin_decode(a.ctx, 1)
    for _ in range(a.steps):
        eng.decode_step()
    eng.sync()
    info = eng.info
    print(json.dumps(info))
    if a.ncu:
        return
    tr = eng.read_trace().astype(np.int64)
    G, L = info["grid"], cfg.n_layers
    t0 = tr[:, 2].min()
    rel = lambda v: (v - t0) / 1e3  # noqa: E731  (us)
    C = info["cluster_size"]
    heads = np.array([(g // C) < cfg.n_heads for g in range(G)])
    out = {"info": info, "kernel_us": float(rel(tr[:, 3].max())),
           "producer_wait_us_med": float(np.median(tr[:, 0]) / CYC),
           "consumer_wait_us_med": float(np.median(tr[:, 1]) / CYC),
           "consumer_wait_us_head_ctas": float(np.median(tr[heads, 1]) / CYC),
           "consumer_wait_us_mlp_ctas": float(np.median(tr[~heads, 1]) / CYC),
           "kv_stage_us_head_ctas": float(np.median(tr[heads, 6]) / CYC),
           "kv_wait_us_head_ctas": float(np.median(tr[heads, 7]) / CYC),
           "att_phase_us_cta0": [float(tr[0, 8 + k]) / CYC for k in range(4)],
           "head_sections_us_per_layer_cta0": {k: float(tr[0, i]) / CYC / L for i, k in
                                                zip(range(8, 16), ["qkv_wait", "kv_append_begin", "att_publish",
                                                                   "att_wait", "att_merge", "qkv_combine_publish",
                                                                   "att_first_stage", "att_other_stages"])},
           "head_phase_us": float(rel(tr[:, 5].max()) - rel(tr[:, 4].min())),
           "layers": []}
    for l in range(L):
        b = 16 + 12 * l
        st, qkv, ctx, end, b1, b2, kv0, pub, pst, fld = (tr[:, b + k] for k in range(10))
        out["layers"].append({
            "start_us": float(rel(st.min())),
            "work_us_med": float(np.median(end - st) / 1e3),
            "work_us_max": float(np.max(end - st) / 1e3),
            "work_us_head_med": float(np.median((end - st)[heads]) / 1e3),
            "work_us_mlp_med": float(np.median((end - st)[~heads]) / 1e3),
            "qkv_us_head_med": float(np.median((qkv - st)[heads]) / 1e3),
            "ctx_us_head_med": float(np.median((ctx - st)[heads]) / 1e3),
            "kv0_us_head_med": float(np.median((kv0 - st)[heads]) / 1e3),
            "att_published_us_head_med": float(np.median((pub - st)[heads]) / 1e3),
            "cluster_reduce_us_med": float(np.median(pst - end) / 1e3),
            "bar1_us_med": float(np.median(b1 - pst) / 1e3),
            "bar1_us_last_arrival_to_release": float((b1.min() - pst.max()) / 1e3),
            "fold_us_med": float(np.median(fld - b1) / 1e3),
            "bar2_us_med": float(np.median(b2 - fld) / 1e3),
            "bar2_us_last_arrival_to_release": float((b2.min() - fld.max()) / 1e3),
            "bar1_wait_us_med": float(np.median(b1 - end) / 1e3),
            "fold_bar2_us_med": float(np.median(b2 - b1) / 1e3),
            "layer_us": float((b2.max() - st.min()) / 1e3),
        })
    lay = out["layers"]
    out["summary"] = {k: float(np.mean([x[k] for x in lay])) for k in lay[0] if k != "start_us"}
    bytes_tok = mean_step_bytes(cfg, a.ctx, 1)
    out["achieved_GBps_this_step"] = bytes_tok / (out["kernel_us"] * 1e-6) / 1e9
    os.makedirs(os.path.dirname(a.out), exist_ok=True)
    with open(a.out, "w") as f:
        json.dump(out, f, indent=1)
    print(json.dumps({k: out[k] for k in out if k not in ("layers",)}, indent=1))


if __name__ == "__main__":
    main()
