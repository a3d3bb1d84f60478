#!/usr/bin/env python
"""Decode throughput of the fused sm_100a GPT-NeoX block (BASELINE.json metric).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]

Workload (BASELINE.json configs[1]): Pythia-2.8B random-init, batch 1,
context 1024, greedy decode in CUDA-graph mode; one *step* = one decoded token
(32 fused layers + final LN + LM head + argmax, one persistent kernel launch).
K timed steps cover positions 1024 .. 1024+K-1.  The per-step working set
(5.65 GB of weights + KV) is ~45x the 126 MB L2, so no L2 flush is needed.

Multi-GPU (torchrun): independent decode streams, one replica per GPU, no
data-path collective ("replicas only"); value = total tokens/s over ranks with
the max-over-ranks device time.

``--impl reference`` times the reference's CPU algorithm (the float64 numpy
port in oracle/, the reference being pure Python) on the host cores, rank 0 only.
"""

from __future__ import annotations

import argparse
import json
import math
import os
import statistics
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

CONTEXT = 1024
METRIC = "decode tokens/s & µs/token (Pythia-2.8B bs=1 ctx1024), % of HBM roofline"
WORKLOAD = "Pythia-2.8B random-init, bs=1, ctx 1024, greedy decode, CUDA graph, 1 launch/token"


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=int(os.environ.get("WORLD_SIZE", "1")),
                    help="GPUs of this node; without a torchrun environment, bench.py spawns the N ranks "
                         "itself (python -m torch.distributed.run, 127.0.0.1)")
    ap.add_argument("--dry-run", action="store_true",
                    help="launch plumbing only (CPU, gloo): ranks, world size, max-over-ranks timing")
    ap.add_argument("--steps", type=int, default=128)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--cpu-seconds", type=float, default=15.0)
    ap.add_argument("--model", default="pythia-2.8b",
                    help="pythia-2.8b (BASELINE configs[1], the headline) or pythia-6.9b (configs[2])")
    ap.add_argument("--context", type=int, default=0, help="KV prefix length (default 1024 / 2048)")
    ap.add_argument("--batch", type=int, default=0,
                    help="batched decode of B sequences (BASELINE configs[3]; default context 4096)")
    ap.add_argument("--tp", action="store_true",
                    help="tensor parallel over the torchrun world (one decode stream; NCCL all-reduce per layer)")
    a = ap.parse_args()
    global CONTEXT, WORKLOAD
    if not a.context:
        a.context = 2048 if a.model == "pythia-6.9b" else (4096 if a.batch else 1024)
    CONTEXT = a.context
    if a.model != "pythia-2.8b" or CONTEXT != 1024:
        name = {"pythia-2.8b": "Pythia-2.8B", "pythia-6.9b": "Pythia-6.9B"}.get(a.model, a.model)
        WORKLOAD = f"{name} random-init, bs=1, ctx {CONTEXT}, greedy decode, CUDA graph, 1 launch/token"
    if a.batch > 1:
        name = {"pythia-2.8b": "Pythia-2.8B", "pythia-6.9b": "Pythia-6.9B"}.get(a.model, a.model)
        WORKLOAD = (f"{name} random-init, batch {a.batch}, ctx {CONTEXT}, greedy decode, CUDA graph "
                    "(tcgen05 hi/lo GEMMs + TMA-tiled attention / LN / GELU kernels)")
    return a


def spawn_ranks(n: int) -> int:
    """`bench.py --gpus N` run directly (no WORLD_SIZE): re-launch this script
    as N ranks under torch.distributed.run on one node, exactly as the driver's
    multi-GPU launch does, and return the launcher's exit code.  Rank 0 prints
    the JSON line."""
    import socket
    import subprocess
    with socket.socket() as sk:
        sk.bind(("127.0.0.1", 0))
        port = sk.getsockname()[1]
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={n}",
           "--master-addr", "127.0.0.1", f"--master-port={port}", os.path.abspath(__file__), *sys.argv[1:]]
    print(f"bench.py: spawning {n} ranks: {' '.join(cmd)}", file=sys.stderr, flush=True)
    return subprocess.call(cmd)


def dist_setup(backend: str = "nccl"):
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world > 1:
        import torch
        import torch.distributed as dist
        if backend == "nccl":
            if torch.cuda.device_count() <= local:
                raise SystemExit(f"rank {rank}: local rank {local} but only {torch.cuda.device_count()} GPU(s)")
            torch.cuda.set_device(local)
            dist.init_process_group("nccl", device_id=torch.device("cuda", local))
        else:
            dist.init_process_group("gloo")
        if rank == 0:
            print(f"bench.py: process group up: backend {dist.get_backend()}, world {dist.get_world_size()}",
                  file=sys.stderr, flush=True)
    return world, rank, local


def run_dry(args, world, rank):
    """Launch plumbing without a GPU: every rank times a tiny CPU loop, the
    max over ranks is reduced like the real bench's device time."""
    from paper_2604_23553_b200.parallel import max_over_ranks
    a = time.perf_counter()
    np.linalg.norm(np.arange(1000.0) * (rank + 1))
    t = max_over_ranks(time.perf_counter() - a)
    if rank == 0:
        print(json.dumps({"dry_run": True, "n_gpus": world, "ranks_reporting": world, "max_rank_seconds": t,
                          "impl": args.impl}), flush=True)


def peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            d = json.load(f)
        return float(d["hbm_gbs"]), "measured"
    except Exception:
        return 6650.0, "fallback"


# ---------------------------------------------------------------------------
# Clock sampling during the timed region (pynvml).

class ClockSampler:
    REASONS = {
        "gpu_idle": 0x1, "applications_clocks_setting": 0x2, "sw_power_cap": 0x4,
        "hw_slowdown": 0x8, "sync_boost": 0x10, "sw_thermal_slowdown": 0x20,
        "hw_thermal_slowdown": 0x40, "hw_power_brake_slowdown": 0x80,
    }

    def __init__(self, index: int):
        self.samples, self.reasons, self.stop = [], set(), threading.Event()
        try:
            import pynvml
            pynvml.nvmlInit()
            self.nv = pynvml
            self.h = pynvml.nvmlDeviceGetHandleByIndex(index)
            self.max = pynvml.nvmlDeviceGetMaxClockInfo(self.h, pynvml.NVML_CLOCK_SM)
        except Exception:
            self.nv = None
            self.max = None

    def _run(self):
        while not self.stop.is_set():
            try:
                self.samples.append(self.nv.nvmlDeviceGetClockInfo(self.h, self.nv.NVML_CLOCK_SM))
                r = self.nv.nvmlDeviceGetCurrentClocksEventReasons(self.h)
                for name, bit in self.REASONS.items():
                    if r & bit and name != "gpu_idle":
                        self.reasons.add(name)
            except Exception:
                pass
            time.sleep(0.005)

    def __enter__(self):
        if self.nv:
            self.t = threading.Thread(target=self._run, daemon=True)
            self.t.start()
        return self

    def __exit__(self, *a):
        if self.nv:
            self.stop.set()
            self.t.join()

    def summary(self):
        if not self.nv or not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": self.max, "reasons": ["unavailable"]}
        return {"sm_mhz": statistics.median(self.samples), "sm_max_mhz": self.max,
                "reasons": sorted(self.reasons), "samples": len(self.samples)}


# ---------------------------------------------------------------------------
# CPU reference path (oracle port of nf/golden.py:189-228), bounded sample.

def cpu_reference(seconds: float, tokens_cap: int | None = None):
    """Time the float64 reference algorithm for the Pythia-2.8B decode token.

    One layer's parameters are shared by all 32 layers (identical arithmetic
    and memory traffic per layer; 20 GB of distinct float64 weights would not
    change the timing).  Returns (tokens_per_s, sample description, threads)."""
    from oracle import neox_oracle as O
    from paper_2604_23553_b200 import preset
    try:  # torchrun pins OMP_NUM_THREADS=1 per rank: give the CPU arm every host core
        from threadpoolctl import threadpool_limits
        threadpool_limits(os.cpu_count())
    except Exception:
        pass
    cfg = preset(MODEL)
    s = O.Shape.of(cfg)
    rng = np.random.default_rng(0)
    p = {}
    for name, shape in O.block_shapes(s).items():
        a = rng.standard_normal(shape)
        p[name] = a / np.sqrt(shape[1]) if len(shape) == 2 else a * 0.02
    p["ln1_gain"] = p["ln2_gain"] = np.ones(s.hidden)
    unembed = rng.standard_normal((s.vocab, s.hidden)) / np.sqrt(s.hidden)
    lnf = (np.ones(s.hidden), np.zeros(s.hidden))
    caches = []
    for _ in range(s.n_layers):
        caches.append(O.KV.of(rng.standard_normal((s.n_heads, CONTEXT, s.d_head)) * 0.5,
                              rng.standard_normal((s.n_heads, CONTEXT, s.d_head)) * 0.5))
    try:
        from threadpoolctl import threadpool_info
        threads = max((i.get("num_threads", 1) for i in threadpool_info()), default=os.cpu_count())
    except Exception:
        threads = os.cpu_count()
    x = rng.standard_normal(s.hidden) * 0.5
    # per-token = sum over the 32 layers + final LN + LM-head GEMV + argmax
    t_tok, done, t0 = [], 0, time.perf_counter()
    while True:
        a = time.perf_counter()
        pos = len(caches[0])
        h = x
        for l in range(s.n_layers):
            h = O.block_step(h, p, caches[l], pos, s)
        lg = unembed @ O.ln_two_pass(h, lnf[0], lnf[1], s.ln_eps)
        O.greedy(lg)
        t_tok.append(time.perf_counter() - a)
        done += 1
        if tokens_cap is not None and done >= tokens_cap:
            break
        if time.perf_counter() - t0 >= seconds:
            break
    per = statistics.mean(t_tok)
    sample = (f"{done} decode token(s) of the float64 numpy port of decoder_block_golden "
              f"(oracle/neox_oracle.block_step) x{s.n_layers} {MODEL} layers (shared layer weights) + "
              f"final LN + LM-head GEMV + argmax, ctx {CONTEXT}, {threads} BLAS threads")
    return 1.0 / per, sample, threads, done


def run_reference(args, world, rank):
    if rank != 0:
        return
    steps, warm = args.steps, args.warmup
    # sized so the arm ends within a few minutes: ~1.3 s/token on 8 cores
    budget = float(os.environ.get("NFB_REF_SECONDS", "150"))
    cpu_reference(0.0, tokens_cap=min(warm, 1) or 1)  # warm-up (page in, BLAS threads)
    tps, sample, threads, done = cpu_reference(budget, tokens_cap=steps)
    if done < steps:
        sample += f" (time-bounded: {done} of the {steps} requested steps)"
    line = {
        "metric": METRIC, "value": tps, "unit": "tokens/s", "n_gpus": world, "steps": done,
        "warmup": warm, "ms_per_step": 1e3 / tps, "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "impl": "reference",
        "config": {"workload": WORKLOAD.replace("CUDA graph, 1 launch/token", "CPU float64"),
                   "context": CONTEXT, "batch": 1, "decode_steps": steps},
        "cpu_baseline": {"value": tps, "unit": "tokens/s", "cores": threads, "kind": "port",
                         "sample": sample},
        "e2e": {"value": tps, "unit": "tokens/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


# ---------------------------------------------------------------------------

def run_batch(args, world, rank, local):
    """BASELINE configs[3]: B sequences at one position (own KV each), one
    token per sequence per step; value = B * steps / time (x world replicas)."""
    import torch
    from paper_2604_23553_b200 import Engine, preset
    from paper_2604_23553_b200.parallel import max_over_ranks
    from paper_2604_23553_b200.perf import mean_batch_step_bytes
    torch.cuda.set_device(local)
    cfg = preset(MODEL)
    B, K, W = args.batch, args.steps, max(args.warmup, 3)
    eng = Engine(cfg, max_seq=CONTEXT + K + W + 8, device=local)
    eng.synth_model(base_seed=1000 * rank)
    eng.batch_init(B)
    eng.batch_kv_synth(CONTEXT, base_seed=7 + rank)
    stream = torch.cuda.ExternalStream(eng.stream, device=torch.device("cuda", local))
    toks0 = [1 + b for b in range(B)]
    eng.batch_begin(CONTEXT, toks0)
    eng.batch_graph_capture()
    eng.batch_step(W)
    eng.sync()
    eng.batch_begin(CONTEXT, toks0)
    start, end = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    if world > 1:
        import torch.distributed as dist
        dist.barrier()
    torch.cuda.synchronize()
    with ClockSampler(local) as clk:
        start.record(stream)
        eng.batch_step(K)
        end.record(stream)
        end.synchronize()
    t = max_over_ranks(start.elapsed_time(end) / 1e3, device=torch.device("cuda", local))
    last = eng.batch_tokens()
    # end to end: one step at a time through the public call + host read of the tokens
    eng.batch_begin(CONTEXT, toks0)
    a = time.perf_counter()
    for _ in range(K):
        eng.batch_step(1)
        last = eng.batch_tokens()
    e2e_t = max_over_ranks(time.perf_counter() - a, device=torch.device("cuda", local))
    if rank != 0:
        return
    bytes_step = mean_batch_step_bytes(cfg, CONTEXT, K, B)
    hbm, kind = peaks()
    achieved = bytes_step / (t / K) / 1e9
    line = {
        "metric": METRIC, "value": world * B * K / t, "unit": "tokens/s", "n_gpus": world, "steps": K,
        "warmup": W, "ms_per_step": t / K * 1e3, "us_per_token": t / K / B * 1e6, "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "f16",
        "data": "synthetic (random-init SplitMix64 weights, synthetic KV prefix per sequence)",
        "config": {"workload": WORKLOAD, "context": CONTEXT, "batch": B, "decode_steps": K,
                   "parallelism": f"replicas x{world}" if world > 1 else "single GPU",
                   "l2": f"no flush: {bytes_step / 1e9:.2f} GB/step working set >> 126 MB L2"},
        "roofline": {"bound": "hbm", "achieved": achieved, "peak": hbm, "unit": "GB/s", "frac": achieved / hbm,
                     "traffic": None, "bytes_per_launch": bytes_step, "peak_kind": kind,
                     "note": "bytes per step (weights once + B x KV); the step is a graph of many launches"},
        "e2e": {"value": world * B * K / e2e_t, "unit": "tokens/s", "h2d_bytes_per_step": 0,
                "d2h_bytes_per_step": 4 * B},
        "gpu_launches": K * (cfg.n_layers * 10 + 5),  # per layer: LN, 4 GEMMs, prep, tiles, combine, GELU, residual
        "clocks": clk.summary(),
        "tokens_tail": [int(x) for x in last[:5]],
    }
    print(json.dumps(line), flush=True)


def run_ours(args, world, rank, local):
    import torch
    from paper_2604_23553_b200 import Engine, mean_step_bytes, preset
    torch.cuda.set_device(local)
    cfg = preset(MODEL)
    K, W = args.steps, max(args.warmup, 3)
    max_seq = CONTEXT + max(K, W, 32) + 8  # 32: the autotune window
    if args.tp:
        # one model sharded over the world: same seeds on every rank
        from paper_2604_23553_b200.parallel import broadcast_bytes
        eng = Engine(cfg, max_seq=max_seq, device=local, tp=(rank, world))
        eng.synth_model(base_seed=0)
        eng.kv_synth_all(CONTEXT, base_seed=7)
        uid = broadcast_bytes(Engine.tp_unique_id() if rank == 0 else None, 128,
                              device=torch.device("cuda", local))
        eng.tp_init(uid)
    else:
        eng = Engine(cfg, max_seq=max_seq, device=local)
        eng.synth_model(base_seed=1000 * rank)
        eng.kv_synth_all(CONTEXT, base_seed=7 + rank)
    stream = torch.cuda.ExternalStream(eng.stream, device=torch.device("cuda", local))
    # pick the static MLP split weight on this box (deterministic afterwards)
    tune = eng.autotune(CONTEXT) if os.environ.get("NFB_AUTOTUNE", "1") != "0" else None

    # warm-up, then restart the decode at position CONTEXT for the timed window
    eng.begin_decode(CONTEXT, token=1)
    eng.graph_capture()
    eng.graph_replay(W)
    eng.sync()
    eng.begin_decode(CONTEXT, token=1)

    def barrier():
        if world > 1:
            import torch.distributed as dist
            dist.barrier()
        torch.cuda.synchronize()

    start, end = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    barrier()
    with ClockSampler(local) as clk:
        start.record(stream)
        eng.graph_replay(K)
        end.record(stream)
        end.synchronize()
    eng.sync()
    t = start.elapsed_time(end) / 1e3
    toks, last = eng.read_tokens(K)
    barrier()
    if world > 1:
        import torch.distributed as dist
        tt = torch.tensor([t], device="cuda")
        dist.all_reduce(tt, op=dist.ReduceOp.MAX)
        t = float(tt.item())

    # end-to-end through the public serving call: host token in, host token out
    eng.begin_decode(CONTEXT, token=1)
    tok = 1
    barrier()
    a = time.perf_counter()
    for _ in range(K):
        tok = eng.step_token(tok)
    e2e_t = time.perf_counter() - a
    if world > 1:
        import torch.distributed as dist
        tt = torch.tensor([e2e_t], device="cuda")
        dist.all_reduce(tt, op=dist.ReduceOp.MAX)
        e2e_t = float(tt.item())

    if rank != 0:
        return
    bytes_step = mean_step_bytes(cfg, CONTEXT, K)
    hbm, kind = peaks()
    ms = t / K * 1e3
    streams = 1 if args.tp else world  # TP: one stream sharded; DP: one stream per GPU
    if args.tp:
        bytes_step /= world  # per-GPU share of the step's weight + KV bytes (roofline of one GPU)
    achieved = bytes_step / (t / K) / 1e9
    traffic = None
    tp = os.path.join(ROOT, "profiles", "ncu_traffic.json")
    if os.path.exists(tp) and MODEL == "pythia-2.8b" and CONTEXT == 1024:
        with open(tp) as f:  # ncu capture of the headline workload only
            traffic = json.load(f).get("dram_bytes_per_launch")
    line = {
        "metric": METRIC,
        "value": streams * K / t,
        "unit": "tokens/s",
        "n_gpus": world,
        "steps": K,
        "warmup": W,
        "ms_per_step": ms,
        "us_per_token": ms * 1e3,
        "higher_is_better": True,
        "scaling": "strong" if args.tp and world > 1 else "weak",
        "vs_baseline": None,
        "dtype": "f16",
        "data": "synthetic (random-init SplitMix64 weights, synthetic KV prefix)",
        "config": {"workload": WORKLOAD, "context": CONTEXT, "batch": 1, "decode_steps": K,
                   "parallelism": (f"tp{world} (NCCL all-reduce per layer)" if args.tp else
                                   f"replicas x{world}" if world > 1 else "single GPU"),
                   "l2": f"no flush: {mean_step_bytes(cfg, CONTEXT, K) / 1e9:.2f} GB/step working set >> 126 MB L2",
                   "autotune": tune},
        "roofline": {"bound": "hbm", "achieved": achieved, "peak": hbm, "unit": "GB/s",
                     "frac": achieved / hbm, "traffic": traffic,
                     "bytes_per_launch": bytes_step, "peak_kind": kind},
        "e2e": {"value": streams * K / e2e_t, "unit": "tokens/s", "h2d_bytes_per_step": 8,
                "d2h_bytes_per_step": 8},
        # fused path: one persistent kernel per token; TP: per layer + LM head + state advance
        "gpu_launches": K * (cfg.n_layers + 2) if args.tp else K,
        "clocks": clk.summary(),
        "tokens_tail": [int(x) for x in toks[-4:]] + [last],
    }
    if world == 1 and not args.no_cpu_baseline:
        tps, sample, threads, _ = cpu_reference(args.cpu_seconds)
        line["cpu_baseline"] = {"value": tps, "unit": "tokens/s", "cores": threads, "kind": "port",
                                "sample": sample}
    print(json.dumps(line), flush=True)


MODEL = "pythia-2.8b"


def main():
    global MODEL
    args = parse()
    MODEL = args.model
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        sys.exit(spawn_ranks(args.gpus))
    if "WORLD_SIZE" in os.environ and int(os.environ["WORLD_SIZE"]) != args.gpus:
        raise SystemExit(f"--gpus {args.gpus} but WORLD_SIZE={os.environ['WORLD_SIZE']}")
    if args.dry_run:
        world, rank, _ = dist_setup("gloo")
        run_dry(args, world, rank)
        if world > 1:
            import torch.distributed as dist
            dist.destroy_process_group()
        return
    if args.impl == "reference":
        world = int(os.environ.get("WORLD_SIZE", "1"))
        rank = int(os.environ.get("RANK", "0"))
        run_reference(args, world, rank)
        return
    world, rank, local = dist_setup()
    if args.batch > 1:  # batch 1 of configs[3] runs on the fused single-sequence kernel
        run_batch(args, world, rank, local)
    else:
        run_ours(args, world, rank, local)
    if world > 1:
        import torch.distributed as dist
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
