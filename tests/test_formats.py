"""On-disk formats: weight manifest + blob, the reference
CLI's golden fixture JSON, the TPOT measurement CSV."""

import json
import os

import numpy as np
import pytest

from oracle import neox_oracle as O
from paper_2604_23553_b200 import ModelConfig, synth_weights
from paper_2604_23553_b200.formats import (fixture_config, format_measurements_csv, parse_measurements_csv)
from paper_2604_23553_b200.weights import load_weights, save_weights

G = os.path.join(os.path.dirname(__file__), "golden")
FIXTURE = os.path.join(G, "cli_golden_h256.json")


def scaled(a, b):
    return float(np.max(np.abs(np.asarray(a) - b)) / np.max(np.abs(b)))


def test_cli_fixture_replays_on_the_oracle():
    """The reference CLI's fixture (made by the reference, tests/golden/make_golden.py)
    replays on the float64 oracle to ~1e-12: pins the fixture format reading."""
    fx = json.load(open(FIXTURE))
    cfg = fixture_config(fx)
    s = O.Shape.of(cfg)
    p = O.synth_block(s, int(fx["seed"]))
    kv = O.KV(s.n_heads, s.d_head)
    outs = [O.block_step(np.asarray(x), p, kv, t, s) for t, x in enumerate(fx["inputs"])]
    assert scaled(outs, np.asarray(fx["outputs"])) < 1e-12
    assert scaled(kv.keys(), np.asarray(fx["cache_keys"])) < 1e-12


def test_weight_files_round_trip(tmp_path):
    cfg = ModelConfig(hidden=64, n_heads=4, d_head=16, n_layers=1, d_mlp=128, rotary_pct=0.25, vocab=32)
    w = synth_weights(cfg, 5)
    save_weights(w, tmp_path / "m.json", tmp_path / "w.bin")
    r = load_weights(tmp_path / "m.json", tmp_path / "w.bin")
    for n in ("qkv_weight", "out_weight", "down_bias"):
        assert np.array_equal(getattr(r, n), getattr(w, n).astype(np.float32).astype(np.float64))


def test_measurement_csv_matches_reference_rules():
    text = format_measurements_csv([(16, 0.9123456, "fused_graph"), (2048, 1.25, "fused")])
    assert text.splitlines()[0] == "seq_len,tpot_ms,variant"
    assert parse_measurements_csv(text) == [(16, 0.9123, "fused_graph"), (2048, 1.25, "fused")]
    with pytest.raises(ValueError, match="unknown variant"):
        format_measurements_csv([(16, 1.0, "b200")])
    with pytest.raises(ValueError, match="bad measurements header"):
        parse_measurements_csv("a,b,c\n1,2,fused\n")
