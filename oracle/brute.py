"""Set-based brute-force enumerator of the sketch definitions (tiny inputs only).

TEST INFRASTRUCTURE ONLY.  Written straight from the plain definition (DESIGN.md "Plain
definition"), independently of usk_oracle.c's streaming update:

  S[i, c]  = argmin_kappa { w_k : idx_i(p_k) = c }   (+inf if the preimage set is empty)
  w'_k     = argmax_rho  { S[i, idx_i(p_k)] : i < M }

kappa orders by (|a|, sign bit) -- Eq. 4's "replace when the absolute value is smaller"
 with ties to the non-negative value (L2); rho orders by (|a|, not sign
bit) -- Eq. 5's max read as max-|.| with the same tie rule.
Values are Python floats (exact for fp32/bf16 inputs).
"""
from __future__ import annotations

import math


def _sign_bit(a: float) -> int:
    return 1 if math.copysign(1.0, a) < 0 else 0


def kappa(a: float):
    return (abs(a), _sign_bit(a))


def rho(a: float):
    return (abs(a), 1 - _sign_bit(a))


def buckets(values, idx, M: int, N: int):
    """values: list of floats; idx[i][k] = bucket of weight k in row i.  Returns S[M][N]."""
    S = []
    for i in range(M):
        row = []
        for c in range(N):
            pre = [values[k] for k in range(len(values)) if idx[i][k] == c]
            row.append(min(pre, key=kappa) if pre else math.inf)
        S.append(row)
    return S


def reconstruct(S, idx, M: int, n: int):
    return [max((S[i][idx[i][k]] for i in range(M)), key=rho) for k in range(n)]
