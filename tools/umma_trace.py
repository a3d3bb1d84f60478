"""Per-CTA phase stamps of the standalone tcgen05 GEMM (nfb_gemm_trace_dev):
where a launch's time goes (setup, first-data latency, streaming, epilogue)."""
import ctypes as C
import json
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2604_23553_b200 import _lib  # noqa: E402

lib = _lib.load()
tr = torch.zeros(148 * 8, dtype=torch.int64, device="cuda")
MODE = os.environ.get("MODE", "flush")  # flush | rotate | warm
for name, M, K in (("qkv", 7680, 2560), ("out", 2560, 2560), ("lm", 50304, 2560)):
    for N in (8, 128):
        W = torch.randn(M, K, device="cuda").half()
        nrot = 4 if MODE == "rotate" else 1
        Wbs = []
        for _ in range(nrot):
            Wb = torch.empty(lib.nfb_gemm_blocked_bytes(M, K) // 2, dtype=torch.float16, device="cuda")
            lib.nfb_gemm_block_weights_dev(M, K, C.c_void_p(W.data_ptr()), C.c_void_p(Wb.data_ptr()), None)
            Wbs.append(Wb)
        flush = torch.empty(int(300e6), dtype=torch.uint8, device="cuda")
        A = torch.randn(N, K, device="cuda").half()
        Y = torch.empty(N, M, device="cuda")
        for it in range(9):
            if MODE == "flush":
                flush.zero_()
            lib.nfb_gemm_trace_dev(C.c_void_p(tr.data_ptr()) if it == 8 else None)
            lib.nfb_gemm_f16_blocked_dev(M, N, K, C.c_void_p(Wbs[it % nrot].data_ptr()), C.c_void_p(A.data_ptr()),
                                         C.c_void_p(Y.data_ptr()), None)
        torch.cuda.synchronize()
        lib.nfb_gemm_trace_dev(None)
        t = tr.cpu().numpy().reshape(148, 8)[:, :7].astype(np.int64)
        t = t[t[:, 0] > 0]
        t0 = t[:, 0].min()
        r = (t - t0) / 1e3
        print(json.dumps({"mode": MODE, "gemm": name, "N": N, "ctas": len(t),
                          **{k: [round(float(np.min(r[:, i])), 2), round(float(np.median(r[:, i])), 2),
                                 round(float(np.max(r[:, i])), 2)]
                             for i, k in enumerate(["start", "setup", "issued", "first_full", "last_mma",
                                                    "epi_done", "exit"])}}))
        tr.zero_()
