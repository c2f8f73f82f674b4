"""Writes tests/golden/hash_vectors.json by calling ONLY oracle/ (never the CUDA path).

These vectors freeze our own hash contract; they are not paper
values.  Run:  python tests/golden/gen_golden.py
"""
import json
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import oracle  # noqa: E402

rng = np.random.default_rng(20250617)
vec = []
for _ in range(64):
    seed = int(rng.integers(0, 2**63))
    layer, t, row = int(rng.integers(0, 224)), int(rng.integers(0, 14336)), int(rng.integers(0, 8))
    p = int(rng.integers(0, 2**32))
    N = int(rng.integers(1, 1 << 20)) if len(vec) % 2 else int(rng.integers(1, 1 << 12))
    vec.append([seed, layer, t, row, p, N, int(oracle.hash_index(0, seed, layer, t, row, p, N))])
out = {"_note": "USK-X (v2: per-row salts, 23-bit short-unit reduction) index vectors written by tests/golden/gen_golden.py from oracle/ only", "vectors": vec}
json.dump(out, open(os.path.join(os.path.dirname(os.path.abspath(__file__)), "hash_vectors.json"), "w"), indent=0)
print("wrote", len(vec))
