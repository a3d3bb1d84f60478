"""Microbenchmark of the tcgen05 batched-projection GEMM (csrc/nfb_umma.cu)
on the C4 shapes: weight GB/s per launch (pre-blocked weights streamed once;
the activations [N][K] are L2-resident).  Weight buffers rotate over > 2x L2
so every launch reads HBM.  The timed call is the steady-state entry
(nfb_gemm_f16_blocked_dev: activation blocking + GEMM + piece sum, three
launches); `us` is per call.  Prints one JSON line per (shape, N).
UMMA_SHAPES=up,qkv UMMA_B=4,16 UMMA_REPS=1 narrow the sweep (for ncu captures)."""

import ctypes as C
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2604_23553_b200 import _lib  # noqa: E402

lib = _lib.load()
SHAPES = {"qkv": (7680, 2560), "out": (2560, 2560), "up": (10240, 2560), "down": (2560, 10240), "lm": (50304, 2560)}
peak = json.load(open(os.path.join(os.path.dirname(__file__), "..", "MEASURED_PEAKS.json")))["hbm_gbs"] \
    if os.path.exists(os.path.join(os.path.dirname(__file__), "..", "MEASURED_PEAKS.json")) else 6650.0
ONLY = os.environ.get("UMMA_SHAPES", "").split(",") if os.environ.get("UMMA_SHAPES") else list(SHAPES)
BATCHES = [int(b) for b in os.environ.get("UMMA_B", "1,4,16,64").split(",")]
REPS = int(os.environ.get("UMMA_REPS", "50"))
for name, (M, K) in SHAPES.items():
    if name not in ONLY:
        continue
    nbuf = max(2, int(300e6 // (M * K * 2)) + 1)
    nb = lib.nfb_gemm_blocked_bytes(M, K)
    Ws = []
    for _ in range(nbuf):
        W = torch.randn(M, K, device="cuda").half()
        Wb = torch.empty(nb // 2, dtype=torch.float16, device="cuda")
        assert lib.nfb_gemm_block_weights_dev(M, K, C.c_void_p(W.data_ptr()), C.c_void_p(Wb.data_ptr()), None) == 0
        Ws.append(Wb)
        del W
    for B in BATCHES:
        N = 2 * B
        A = torch.randn(N, K, device="cuda").half()
        Y = torch.empty(N, M, device="cuda")
        st = torch.cuda.current_stream().cuda_stream

        def run(i):
            rc = lib.nfb_gemm_f16_blocked_dev(M, N, K, C.c_void_p(Ws[i % nbuf].data_ptr()), C.c_void_p(A.data_ptr()),
                                      C.c_void_p(Y.data_ptr()), C.c_void_p(st))
            assert rc == 0

        for i in range(5):
            run(i)
        reps = REPS
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize()
        e0.record()
        for i in range(reps):
            run(i)
        e1.record()
        torch.cuda.synchronize()
        t = e0.elapsed_time(e1) / reps * 1e-3
        gbs = M * K * 2 / t / 1e9
        print(json.dumps({"gemm": name, "M": M, "K": K, "B": B, "N": N, "us": t * 1e6, "weight_GBps": gbs,
                          "frac": gbs / peak, "tflops": 2 * M * N * K / t / 1e12}), flush=True)
