#!/usr/bin/env python
"""Measured B200 TPOT in the reference's measurement CSV (seq_len,tpot_ms,variant;
nf/perfmodel.py:337-398): Pythia-2.8B, 5-token prompt, N decoded tokens (the
paper's "decode tokens" axis, nf/perfmodel.py:51), eager launches ("fused")
and CUDA-graph replay ("fused_graph").  Feed it to the reference's
`neoxfuse calibrate --measurements FILE` to fit B200 parameters.

    python tools/tpot_csv.py --out profiles/r01_tpot_pythia28b_b200.csv
"""
import argparse
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from paper_2604_23553_b200 import Engine, preset  # noqa: E402
from paper_2604_23553_b200.formats import format_measurements_csv  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--out", default=os.path.join(ROOT, "profiles", "tpot_b200.csv"))
    ap.add_argument("--lens", default="16,32,64,128,256,512,1024,2048")
    a = ap.parse_args()
    import torch
    lens = [int(x) for x in a.lens.split(",")]
    prompt = 5
    eng = Engine(preset("pythia-2.8b"), max_seq=prompt + max(lens) + 8)
    eng.synth_model(0)
    eng.kv_synth_all(prompt, 7)
    stream = torch.cuda.ExternalStream(eng.stream)
    rows = []
    for variant in ("fused", "fused_graph"):
        for n in lens:
            eng.begin_decode(prompt, token=1)
            if variant == "fused_graph":
                eng.graph_capture()
            start, end = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            start.record(stream)
            if variant == "fused_graph":
                eng.graph_replay(n)
            else:
                for _ in range(n):
                    eng.decode_step()
            end.record(stream)
            end.synchronize()
            ms = start.elapsed_time(end) / n
            rows.append((n, ms, variant))
            print(f"{variant:12s} n={n:5d} tpot {ms:.4f} ms (wall {(time.perf_counter() - t0) / n * 1e3:.4f})")
    os.makedirs(os.path.dirname(a.out), exist_ok=True)
    with open(a.out, "w") as f:
        f.write(format_measurements_csv(rows))
    print("wrote", a.out)


if __name__ == "__main__":
    main()
