#!/usr/bin/env python
"""Where the end-to-end serving step loses time against graph replay (C2):
back-to-back replays, one replay + host sync per token, and the serving call
(token H2D + replay + argmax D2H + sync) per token.  Prints us/token each."""
import os
import sys
import time

if "--torch" in sys.argv:
    import torch
    torch.cuda.init()

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2604_23553_b200 import Engine, preset  # noqa: E402

K, CTX = 128, 1024
eng = Engine(preset("pythia-2.8b"), max_seq=CTX + 2 * K + 8)
eng.synth_model(0)
eng.kv_synth_all(CTX, 7)
if "--autotune" in sys.argv:
    print("autotune", eng.autotune(CTX))
eng.begin_decode(CTX, token=1)
eng.graph_capture()
eng.graph_replay(8)
eng.sync()
res = {}
for name in ("replay_back_to_back", "replay_sync_each", "step_token", "replay_back_to_back"):
    eng.begin_decode(CTX, token=1)
    eng.sync()
    a = time.perf_counter()
    if name == "replay_back_to_back":
        eng.graph_replay(K)
        eng.sync()
    elif name == "replay_sync_each":
        for _ in range(K):
            eng.graph_replay(1)
            eng.sync()
    else:
        tok = 1
        for _ in range(K):
            tok = eng.step_token(tok)
    res[name] = round((time.perf_counter() - a) / K * 1e6, 1)
print(res)
