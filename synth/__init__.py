"""Seeded synthetic inputs shared by the oracle tests, the GPU parity tests and bench.py.

This module holds NONE of the method's arithmetic (no hashing, no sketching, no allocation,
no importance metric): only random draws, edge-case matrices and model shapes.  The recipe
is stated in DESIGN.md "Input recipe":

* weights: bf16 = RNE(0.02 * z), z ~ N(0, 1) (Gaussian, as in Appendix B's setting and
  SPEC's standard-normal tests; 0.02 is a Llama-like scale, not a paper number);
  fp32 weights for config 1 are z ~ N(0, 1).
* activations for saliency: a_kj = sigma_j z_kj, sigma_j = exp(0.5 xi_j), 1% outlier channels x20.
* decode inputs x ~ N(0, 1); prefill X ~ N(0, 1) bf16.
* seeds: seed = 1000 * cfg + 7 * block + k  (k = index of the linear in the block).
"""
from __future__ import annotations

import numpy as np

# --------------------------------------------------------------------------- model shapes
# Llama-3.2-1B: hidden 2048, 8 KV heads x 64, MLP 8192, 16 blocks.  Llama-3-8B: hidden 4096,
# 8 KV heads x 128, MLP 14336, 32 blocks.  [out_features, in_features] per linear, canonical
# order q, k, v, o, gate, up, down (layer id = 7 * block + k).
LINEAR_NAMES = ("q", "k", "v", "o", "gate", "up", "down")


def llama_block(hidden, kv, mlp):
    return [(hidden, hidden), (kv, hidden), (kv, hidden), (hidden, hidden), (mlp, hidden), (mlp, hidden),
            (hidden, mlp)]


def llama32_1b_shapes():
    return llama_block(2048, 512, 8192) * 16


def llama3_8b_shapes():
    return llama_block(4096, 1024, 14336) * 32


def mlp_block_1b_shapes():
    return [(8192, 2048), (8192, 2048), (2048, 8192)]


def seed_for(cfg: int, block: int, k: int) -> int:
    return 1000 * cfg + 7 * block + k


# --------------------------------------------------------------------------- bf16 bits
def f32_to_bf16_bits(a: np.ndarray) -> np.ndarray:
    """Round-to-nearest-even fp32 -> bf16 bit patterns (uint16).  Inputs must be finite."""
    b = np.ascontiguousarray(a, dtype=np.float32).view(np.uint32).astype(np.uint64)
    rounded = (b + 0x7FFF + ((b >> 16) & 1)) >> 16
    return rounded.astype(np.uint16)


def bf16_bits_to_f32(b: np.ndarray) -> np.ndarray:
    return (np.asarray(b).astype(np.uint32) << np.uint32(16)).view(np.float32)


# --------------------------------------------------------------------------- CPU generators
def weights_bf16(out: int, inn: int, seed: int, scale: float = 0.02) -> np.ndarray:
    rng = np.random.default_rng(seed)
    z = rng.standard_normal((out, inn), dtype=np.float32)
    return f32_to_bf16_bits(z * np.float32(scale))


def weights_f32(out: int, inn: int, seed: int, scale: float = 1.0) -> np.ndarray:
    rng = np.random.default_rng(seed)
    return (rng.standard_normal((out, inn), dtype=np.float32) * np.float32(scale)).astype(np.float32)


def vector(n: int, seed: int, T: int = 1) -> np.ndarray:
    rng = np.random.default_rng(seed)
    return rng.standard_normal((T, n), dtype=np.float32)


def activations(N: int, d: int, seed: int) -> np.ndarray:
    """Calibration activations [N, d]: per-channel log-normal scale, 1% outlier channels x20."""
    rng = np.random.default_rng(seed)
    sigma = np.exp(0.5 * rng.standard_normal(d)).astype(np.float32)
    n_out = max(1, d // 100)
    sigma[rng.choice(d, n_out, replace=False)] *= 20.0
    return (rng.standard_normal((N, d), dtype=np.float32) * sigma[None, :]).astype(np.float32)


def saliency_like(d: int, seed: int) -> np.ndarray:
    """Positive per-input-dim scores with the shape of an Eq. 7 profile (log-normal, 1% x400)."""
    rng = np.random.default_rng(seed)
    s = np.exp(rng.standard_normal(d)).astype(np.float32)
    n_out = max(1, d // 100)
    s[rng.choice(d, n_out, replace=False)] *= 400.0
    return s


def edge_matrix_f32(kind: str, out: int, inn: int, seed: int = 0) -> np.ndarray:
    """Degenerate inputs for the bit-exact tests."""
    rng = np.random.default_rng(seed)
    if kind == "all_equal":
        return np.full((out, inn), 0.375, dtype=np.float32)
    if kind == "pm_pairs":  # +x / -x ties everywhere
        v = rng.choice(np.array([0.25, 0.5, 1.0], np.float32), size=(out, inn))
        sgn = rng.choice(np.array([-1.0, 1.0], np.float32), size=(out, inn))
        return (v * sgn).astype(np.float32)
    if kind == "zeros":  # +0 and -0
        return np.where(rng.random((out, inn)) < 0.5, np.float32(0.0), np.float32(-0.0)).astype(np.float32)
    if kind == "subnormal":
        m = rng.integers(1, 1 << 23, size=(out, inn), dtype=np.uint32)
        s = rng.integers(0, 2, size=(out, inn), dtype=np.uint32) << np.uint32(31)
        return (m | s).view(np.float32)
    if kind == "outlier":
        w = rng.standard_normal((out, inn), dtype=np.float32)
        w[out // 2, inn // 3] = np.float32(1e30)
        return w
    if kind == "mixed":  # ties, zeros, subnormals and normals together
        w = rng.standard_normal((out, inn), dtype=np.float32)
        r = rng.random((out, inn))
        w[r < 0.1] = 0.0
        w[(r >= 0.1) & (r < 0.2)] = -0.0
        w[(r >= 0.2) & (r < 0.35)] = np.float32(0.5)
        w[(r >= 0.35) & (r < 0.5)] = np.float32(-0.5)
        sub = (r >= 0.5) & (r < 0.6)
        w[sub] = np.array([1e-40], np.float32)[0] * np.sign(rng.standard_normal(int(sub.sum()))).astype(np.float32)
        return w.astype(np.float32)
    raise ValueError(kind)


def edge_matrix_bf16(kind: str, out: int, inn: int, seed: int = 0) -> np.ndarray:
    if kind == "subnormal":
        rng = np.random.default_rng(seed)
        m = rng.integers(1, 1 << 7, size=(out, inn), dtype=np.uint16)
        s = rng.integers(0, 2, size=(out, inn), dtype=np.uint16) << np.uint16(15)
        return (m | s).astype(np.uint16)
    return f32_to_bf16_bits(edge_matrix_f32(kind, out, inn, seed))


# --------------------------------------------------------------------------- device generators
def torch_weights_bf16(out: int, inn: int, seed: int, device, scale: float = 0.02):
    """Same recipe drawn with a seeded torch generator on `device` (bench / full-size parity)."""
    import torch
    gen = torch.Generator(device=device)
    gen.manual_seed(seed)
    z = torch.randn((out, inn), generator=gen, device=device, dtype=torch.float32)
    return (z * scale).to(torch.bfloat16)


def torch_vector(n: int, seed: int, device, dtype, T: int = 1):
    import torch
    gen = torch.Generator(device=device)
    gen.manual_seed(seed)
    return torch.randn((T, n), generator=gen, device=device, dtype=torch.float32).to(dtype)
