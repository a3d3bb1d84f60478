"""On-disk formats around the decode path.

* Weight files: the reference's manifest (JSON) + raw float32 blob
  (``save_weights`` / ``load_weights``, nf/weights.py:97-129) loaded straight
  into a device context (``load_block_weights``): fp16 RNE on upload, the
  kernel's layouts (transposed W_out / W_down) built by the C library.
* Golden fixtures: the reference CLI's JSON (``neoxfuse golden``,
  nf/cli.py:343-397 -- model, seed, inputs, outputs, cache) replayed through
  the fused sm_100a block (``replay_golden_fixture``).
* TPOT measurements: the reference's ``seq_len,tpot_ms,variant`` CSV
  (nf/perfmodel.py:337-398) written from measured B200 decode times
  (``tools/tpot_csv.py``) so its ``calibrate`` can fit B200 parameters.
"""

from __future__ import annotations

import csv
import io
import json
from dataclasses import dataclass
from pathlib import Path

import numpy as np

from .config import ModelConfig
from .weights import load_weights

MEASUREMENT_HEADER = ("seq_len", "tpot_ms", "variant")
# the reference's variant names (nf/perfmodel.py:342-348)
VARIANTS = ("baseline", "fused", "fused_graph", "attention_only", "mlp_down_only")


def load_block_weights(engine, layer: int, manifest_path, blob_path) -> None:
    """Reference weight files of one block -> device context layer."""
    w = load_weights(manifest_path, blob_path)
    w.validate(engine.cfg)
    engine.set_block_weights(layer, w)


def fixture_config(fx: dict) -> ModelConfig:
    m = fx["model"]
    return ModelConfig(hidden=m["hidden"], n_heads=m["n_heads"], d_head=m["d_head"], n_layers=m["n_layers"],
                       d_mlp=m["d_mlp"], rotary_pct=m["rotary_pct"], vocab=m["vocab"], ln_eps=m["ln_eps"],
                       theta_base=m["theta_base"], parallel_residual=m["parallel_residual"])


@dataclass
class FixtureReplay:
    outputs: np.ndarray       # [steps, hidden] from the kernel
    keys: np.ndarray          # [heads, steps, d_head] cache after the replay
    values: np.ndarray
    output_error: float       # scaled max error vs the fixture (nf/verify.py:103-104)
    cache_error: float


def _scaled(a, b) -> float:
    b = np.asarray(b, np.float64)
    return float(np.max(np.abs(np.asarray(a, np.float64) - b)) / max(np.max(np.abs(b)), 1e-30))


def replay_golden_fixture(path_or_dict, manifest=None, blob=None, device: int = 0) -> FixtureReplay:
    """Replay a ``neoxfuse golden`` fixture: same weights (seeded synthesis or
    the given weight files), same inputs, empty cache, one fused block step
    per input on the GPU; returns the outputs and their error vs the fixture."""
    from .engine import Engine
    fx = path_or_dict if isinstance(path_or_dict, dict) else json.loads(Path(path_or_dict).read_text())
    cfg = fixture_config(fx)
    xs = np.asarray(fx["inputs"], np.float64)
    with Engine(cfg, max_seq=len(xs) + 8, gelu=fx.get("gelu", "tanh"), device=device) as eng:
        if manifest and blob:
            load_block_weights(eng, 0, manifest, blob)
        elif str(fx.get("weights_source", "")).startswith("synthesized"):
            eng.synth_block_weights(0, int(fx["seed"]))
        else:
            raise ValueError("fixture weights come from files: pass manifest= and blob=")
        outs = np.array([eng.block_step(0, t, xs[t]) for t in range(len(xs))])
        k, v = eng.kv_read(0, 0, len(xs))
    want_k, want_v = np.asarray(fx["cache_keys"]), np.asarray(fx["cache_values"])
    return FixtureReplay(outs, k, v, _scaled(outs, fx["outputs"]),
                         max(_scaled(k, want_k), _scaled(v, want_v)))


def format_measurements_csv(rows) -> str:
    """rows: (seq_len, tpot_ms, variant) -> the reference's measurement CSV."""
    out = io.StringIO()
    w = csv.writer(out, lineterminator="\n")
    w.writerow(MEASUREMENT_HEADER)
    for seq, tpot, variant in rows:
        if variant not in VARIANTS:
            raise ValueError(f"unknown variant {variant!r} (known: {', '.join(sorted(VARIANTS))})")
        if int(seq) < 1 or not float(tpot) > 0:
            raise ValueError("out-of-range values")
        w.writerow((int(seq), f"{float(tpot):.4f}", variant))
    return out.getvalue()


def parse_measurements_csv(text: str) -> list[tuple[int, float, str]]:
    """Restatement of the reference parser's rules (nf/perfmodel.py:355-386)."""
    reader = csv.reader(io.StringIO(text))
    header = tuple(next(reader, ()))
    if header != MEASUREMENT_HEADER:
        raise ValueError(f"bad measurements header {header!r}, expected {MEASUREMENT_HEADER!r}")
    rows = []
    for lineno, row in enumerate(reader, start=2):
        if not row:
            continue
        if len(row) != 3:
            raise ValueError(f"line {lineno}: expected 3 columns, got {len(row)}")
        seq, tpot, variant = int(row[0]), float(row[1]), row[2]
        if variant not in VARIANTS:
            raise ValueError(f"line {lineno}: unknown variant {variant!r}")
        if seq < 1 or tpot <= 0:
            raise ValueError(f"line {lineno}: out-of-range values")
        rows.append((seq, tpot, variant))
    if not rows:
        raise ValueError("measurements table has no data rows")
    return rows
