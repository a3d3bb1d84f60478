#!/usr/bin/env python
"""Per-stage timeline of one layer (lrel = L/2) of a traced decode step:
consumer wait / work per ring stage and producer push times, for a few CTAs.

    python tools/trace_stages.py [--ctas 0,1,100] [--out gpurun_out/stages.json]
"""
import argparse
import json
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from paper_2604_23553_b200 import Engine, preset  # noqa: E402

NAMES = {1: "QKV", 2: "KV", 3: "WO", 4: "UP", 5: "DOWN", 6: "SYNC", 7: "END", 8: "LM", 9: "HEND", 10: "AQKV", 11: "HKV"}
MAXS = 64


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--preset", default="pythia-2.8b")
    ap.add_argument("--ctx", type=int, default=1024)
    ap.add_argument("--ctas", default="0,1,100,147")
    ap.add_argument("--out", default=os.path.join(ROOT, "gpurun_out", "stages.json"))
    a = ap.parse_args()
    cfg = preset(a.preset)
    eng = Engine(cfg, max_seq=a.ctx + 16)
    eng.synth_model(0)
    eng.kv_synth_all(a.ctx, 7)
    eng.set_option("trace", True)
    eng.begin_decode(a.ctx, 1)
    for _ in range(3):
        eng.decode_step()
    eng.sync()
    tr = eng.read_trace().astype(np.int64)
    L = cfg.n_layers
    lrel = L // 2
    base = 16 + 12 * L
    res = {}
    for g in [int(x) for x in a.ctas.split(",")]:
        row = tr[g]
        GHZ = 1.965  # clock64 ticks -> ns at the max SM clock (bench shows it holds)
        cons = row[base:base + 4 * MAXS].reshape(MAXS, 4)
        prod = row[base + 4 * MAXS:base + 6 * MAXS].reshape(MAXS, 2)
        stages = []
        t0 = cons[0][0]
        for i in range(MAXS):
            b, w, r, code = cons[i]
            if b == 0:
                break
            typ = int(code & 0xff)
            stages.append({"i": i, "type": NAMES.get(typ, typ), "n": int((code >> 8) & 0xffffff),
                           "flags": int((code >> 32) & 0xff), "head": int((code >> 40) & 0xffffff),
                           "t_begin_us": (b - t0) / GHZ / 1e3, "wait_us": (w - b) / GHZ / 1e3,
                           "work_us": (r - w) / GHZ / 1e3 if r else None})
        pushes = [{"i": i, "t_begin_us": (pb - t0) / GHZ / 1e3, "wait_issue_us": (pe - pb) / GHZ / 1e3}
                  for i, (pb, pe) in enumerate(prod) if pb]
        res[g] = {"stages": stages, "pushes": pushes}
        print(f"--- CTA {g}")
        for s in stages:
            print(f"  {s['i']:2d} {s['type']:>5} n={s['n']:3d} f={s['flags']} t={s['t_begin_us']:7.2f} "
                  f"wait={s['wait_us']:6.2f} work={s['work_us'] if s['work_us'] is None else round(s['work_us'], 3)}")
        tot = {}
        for s in stages:
            k = s["type"]
            a0 = tot.setdefault(k, [0, 0.0, 0.0])
            a0[0] += 1
            a0[1] += s["wait_us"]
            a0[2] += s["work_us"] or 0.0
        print("  by type (count, wait us, work us):", {k: (v[0], round(v[1], 2), round(v[2], 2)) for k, v in tot.items()})
        pw = [p["wait_issue_us"] for p in pushes]
        print(f"  producer: {len(pushes)} pushes, first at {pushes[0]['t_begin_us'] if pushes else None}, "
              f"empty-wait+issue total {sum(pw):.2f} us")
    os.makedirs(os.path.dirname(a.out), exist_ok=True)
    json.dump(res, open(a.out, "w"), indent=1)


if __name__ == "__main__":
    main()
