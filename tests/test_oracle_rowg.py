"""Pin of ROW units spanning g > 1 input dims (DESIGN.md 2.1 / ledger L7; "each
row ... an independent AbsMaxMin sketch instance" of 1e4-1e5 weights): unit t of a layer holds the
input dims j in [t g, (t + 1) g) and weight (o, j) sits at position p = (j - t g) out + o.  The
positions are re-derived here from that sentence and the buckets / reconstruction enumerated by the
set-based brute force (oracle/brute.py), independently of usk_oracle.c's unit_pos."""
import math

import numpy as np
import pytest

import synth
from oracle import brute


@pytest.mark.parametrize("dtype,g,M,bpw", [(1, 4, 3, 4.0), (0, 2, 2, 8.0), (1, 3, 1, 2.0)])
def test_row_units_g_gt_1_match_brute_force(orc, dtype, g, M, bpw):
    out, inn = 16, 12
    pl = orc.plan([(out, inn)], bpw, M=M, dtype=dtype, g=g, seed=0xC0FFEE)
    W = synth.edge_matrix_bf16("mixed", out, inn, seed=6) if dtype == 1 else \
        synth.edge_matrix_f32("mixed", out, inn, seed=6)
    sk = orc.build_model(pl, [W])
    Wp = orc.reconstruct_rows(pl, sk, 0)
    bits = W.astype(np.uint32) if dtype == 1 else W.view(np.uint32)
    shift = 16 if dtype == 1 else 0
    assert len(pl.ncols) == inn // g
    for t in range(inn // g):
        N, off = int(pl.ncols[t]), int(pl.offsets[t])
        members = [(o, j) for j in range(t * g, (t + 1) * g) for o in range(out)]
        pos = np.array([(j - t * g) * out + o for o, j in members], np.uint32)
        vals = [float(orc.value_of(np.array([bits[o, j]]), dtype)[0]) for o, j in members]
        idx = orc.hash_indices(orc.HASH_X, pl.seed, 0, t, M, pos, N)
        S = brute.buckets(vals, idx, M, N)
        inf = 0x7F80 if dtype else 0x7F800000
        want = [inf if math.isinf(v) else int(orc.bits_of(np.array([v], np.float32), 0)[0]) >> shift
                for row in S for v in row]
        np.testing.assert_array_equal(sk[off:off + M * N].astype(np.uint32), np.array(want, np.uint32))
        rec = brute.reconstruct(S, idx, M, len(members))
        for (o, j), v in zip(members, rec):
            assert int(Wp[o, j]) == int(orc.bits_of(np.array([v], np.float32), 0)[0]) >> shift, (t, o, j)
