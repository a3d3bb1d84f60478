#!/usr/bin/env python
"""A few eager batched decode steps (for an ncu launch list of the batch path)."""
import argparse, os, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2604_23553_b200 import Engine, preset  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--batch", type=int, default=16)
ap.add_argument("--ctx", type=int, default=4096)
ap.add_argument("--steps", type=int, default=2)
a = ap.parse_args()
eng = Engine(preset("pythia-2.8b"), max_seq=a.ctx + a.steps + 8)
eng.synth_model(0)
eng.batch_init(a.batch)
eng.batch_kv_synth(a.ctx, 7)
eng.batch_begin(a.ctx, list(range(1, a.batch + 1)))
eng.batch_step(a.steps)
eng.sync()
print("ok")
