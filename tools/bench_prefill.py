#!/usr/bin/env python
"""Prefill throughput (reference prefill_attention_tiled,
nf/golden.py:234-265): a T-token prompt through all layers of Pythia-2.8B on
the batched kernels (chunks of max_batch rows, causal attention over the one
cache, K/V appended), timed with CUDA events on the context stream after a
warm-up prefill.  Prints one JSON line per (T, chunk)."""
import argparse
import json
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2604_23553_b200 import Engine, preset  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--tokens", default="512,1024,2048")
    ap.add_argument("--chunks", default="32,64,128")
    a = ap.parse_args()
    cfg = preset("pythia-2.8b")
    Ts = [int(t) for t in a.tokens.split(",")]
    rng = np.random.default_rng(0)
    for ch in [int(c) for c in a.chunks.split(",")]:
        for T in Ts:
            eng = Engine(cfg, max_seq=T + ch + 8)
            eng.synth_model(0)
            eng.batch_init(ch)
            st = torch.cuda.ExternalStream(eng.stream)
            xs = rng.standard_normal((T, cfg.hidden)).astype(np.float32) * 0.5
            eng.prefill(0, xs[:ch])  # warm-up chunk (plans, blocked weights); the timed prompt follows it
            s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            torch.cuda.synchronize()
            s.record(st)
            out = eng.prefill(ch, xs)
            e.record(st)
            e.synchronize()
            ms = s.elapsed_time(e)
            print(json.dumps({"prefill_tokens": T, "chunk_rows": ch, "ms": ms, "tokens_per_s": T / ms * 1e3,
                              "finite": bool(np.isfinite(out).all()),
                              "note": "host->device prompt copy and per-chunk host sync included"}), flush=True)
            eng.close()

if __name__ == "__main__":
    main()
