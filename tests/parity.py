"""The parity comparator every GPU test uses (test infrastructure).

* North-star bar (BASELINE.json): scaled error max|a-b| / max|b| <= 2e-2 on
  per-layer hidden states and logits (nf/verify.py:103-104 convention).
* That bar alone cannot catch real bugs: a block output is dominated by its
  residual input x, so a dropped head or a missing fresh token moves it by
  only ~1e-2.  Every check therefore also asserts
    - the regression guard: scaled error <= TIGHT_BLOCK (2e-5) for one block
      step, TIGHT (1e-4) through many layers (the kernel sits at ~1e-6 per
      block: fp32 accumulation against the float64 oracle on the same fp16
      weights / fp16 KV store), and
    - the residual-free delta: scaled(out - x, want - x) <= 2e-2.
  tests/test_parity_comparator.py proves the comparator rejects mutated
  oracles (the nf/verify.py:67-69 "the harness can fail" pattern).
"""

import numpy as np

TOL = 2e-2
TIGHT = 1e-4        # multi-layer hidden states / logits
TIGHT_BLOCK = 2e-5  # one block step (measured ~1e-6 at C1)


def scaled(a, b) -> float:
    a = np.asarray(a, np.float64)
    b = np.asarray(b, np.float64)
    return float(np.max(np.abs(a - b)) / max(np.max(np.abs(b)), 1e-30))


def check(got, want, x=None, tight=TIGHT_BLOCK, what="") -> dict:
    """Assert the three bars; returns the measured errors."""
    e = {"scaled": scaled(got, want)}
    assert e["scaled"] <= TOL, f"{what}: scaled error {e['scaled']:.3e} > north-star bar {TOL}"
    assert e["scaled"] <= tight, f"{what}: scaled error {e['scaled']:.3e} > regression guard {tight:.0e}"
    if x is not None:
        x = np.asarray(x, np.float64)
        e["delta"] = scaled(np.asarray(got, np.float64) - x, np.asarray(want, np.float64) - x)
        assert e["delta"] <= TOL, f"{what}: residual-free delta error {e['delta']:.3e} > {TOL}"
    return e
