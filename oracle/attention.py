"""fp64 attention forward -- TEST INFRASTRUCTURE (F4 workload check).

Same import rule as the rest of ``oracle/``: only ``tests/``, ``smoke()`` and
``bench.py``'s CPU legs use it; it imports nothing from the product path.

The F4 drift study runs an attention
forward kernel ("attn_fwd", fp16, B=2, H=16, S=4096, D=128) under two tile
configurations and compares their outputs with K2.  This module is the plain
definition the kernel approximates, so that the study can show both configs
are equally close to the exact result while differing from each other:

    O = softmax(sm_scale * Q K^T) V,   softmax over the key axis,

computed in fp64 from the fp16 inputs (each converted exactly), rows on
request.  The max subtraction is the textbook one-pass stabilisation; it does
not change the exact value.  Pins: tests/test_oracle_attention.py (uniform
scores -> column mean of V, a dominant key -> that V row, joint key/value
permutation invariance, convex-hull bounds, sm_scale = 0).
"""
from __future__ import annotations

import numpy as np


def attention_rows(q: np.ndarray, k: np.ndarray, v: np.ndarray, rows, sm_scale: float) -> np.ndarray:
    """Exact (fp64) attention output rows of one head.

    q, k, v: [S, D] arrays (any float dtype, converted exactly to fp64);
    rows: query row indices; returns [len(rows), D] fp64."""
    q64 = np.asarray(q, dtype=np.float64)[np.asarray(rows)]
    k64 = np.asarray(k, dtype=np.float64)
    v64 = np.asarray(v, dtype=np.float64)
    scores = (q64 @ k64.T) * float(sm_scale)                 # [R, S]
    scores -= scores.max(axis=1, keepdims=True)
    w = np.exp(scores)
    w /= w.sum(axis=1, keepdims=True)                        # softmax over keys
    return w @ v64                                           # [R, D]
