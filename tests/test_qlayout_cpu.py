"""CPU checks of tests/qlayout.py (the query layout of include/usk.h, written from its text) on
oracle sketches: pack / unpack is a bijection of the unit-major cells, padding is 0, sizes follow
the header's formula; and the library exports the query-layout entry fields (no GPU needed)."""
import numpy as np

import qlayout
import synth


def test_pack_unpack_roundtrip(orc):
    shapes = [(200, 72), (130, 264), (96, 512)]
    opl = orc.plan(shapes, 0.5, M=3, dtype=orc.BF16, hash_kind=orc.HASH_XG, seed=3)
    Ws = [synth.weights_bf16(o, i, 40 + k) for k, (o, i) in enumerate(shapes)]
    sk = orc.build_model(opl, Ws)
    for l, (o, i) in enumerate(shapes):
        u0, u1 = opl.layer_units(l)
        offs = opl.offsets[u0:u1 + 1]
        q = qlayout.pack_layer(sk[offs[0]:], offs - offs[0], opl.ncols[u0:u1], opl.nrows[u0:u1], 3)
        mx, sizes, cw = qlayout.layer_geometry(opl.ncols[u0:u1], 3)
        assert q.size * 2 == sum(sizes) and len(mx) == (i + cw - 1) // cw
        cells, pad_ok = qlayout.unpack_layer(q, offs, opl.ncols[u0:u1], opl.nrows[u0:u1], 3)
        np.testing.assert_array_equal(cells, sk[offs[0]:offs[-1]])
        assert pad_ok
        # rho16 is a bijection of the bf16 bits ordered by (|w|, non-negative first)
        b = np.arange(1 << 16, dtype=np.uint16)
        r = qlayout.rho16(b)
        assert np.unique(r).size == 1 << 16
        np.testing.assert_array_equal(qlayout.unrho16(r), b)


def test_class_order_roundtrip(orc):
    """Class-ordered layers (ledger L34): pack / unpack is a bijection, chunks never straddle a class,
    every unit's cells sit at its query position, and every chunk fits shared memory."""
    shapes = [(512, 1024), (300, 2048), (2048, 512)]
    sal = [synth.saliency_like(i, 90 + k) for k, (o, i) in enumerate(shapes)]
    for crows in (None, (3, 3, 2, 2)):
        opl = orc.plan(shapes, 0.5, M=3, dtype=orc.BF16, hash_kind=orc.HASH_XG, seed=9, saliency=sal, C=4,
                       class_rows=crows)
        Ws = [synth.weights_bf16(o, i, 95 + k) for k, (o, i) in enumerate(shapes)]
        sk = orc.build_model(opl, Ws)
        for l in range(len(shapes)):
            u0, u1 = opl.layer_units(l)
            nc, nr, cl = opl.ncols[u0:u1], opl.nrows[u0:u1], opl.cls[u0:u1]
            offs = opl.offsets[u0:u1 + 1]
            ch, order = qlayout.chunks(nc, nr, 3, cl)
            assert [int(cl[8 * g]) for g in order] == sorted(int(cl[8 * g]) for g in order)
            for (q0, n, cw, mx, mr) in ch:
                units = [8 * order[(q0 + s) // 8] + (q0 + s) % 8 for s in range(n)]
                assert len({int(cl[u]) for u in units}) == 1 and n <= cw
                assert mr * mx * 2 * cw <= qlayout.SMEM_CAP
            q = qlayout.pack_layer(sk[offs[0]:], offs - offs[0], nc, nr, 3, cl)
            cells, pad_ok = qlayout.unpack_layer(q, offs, nc, nr, 3, cl)
            np.testing.assert_array_equal(cells, sk[offs[0]:offs[-1]])
            assert pad_ok
            for t in (0, len(nc) // 2 + 3, len(nc) - 1):
                np.testing.assert_array_equal(qlayout.unit_cells(q, nc, nr, t, 3, cl), sk[offs[t]:offs[t + 1]])


def test_abi_declares_query_layout():
    import re, os
    h = open(os.path.join(os.path.dirname(__file__), "..", "include", "usk.h")).read()
    assert re.search(r"USK_LAYOUT_QUERY\s*=\s*1", h) and re.search(r"USK_HASH_XG\s*=\s*2", h)
    assert "qbyte_begin" in h and "int32_t layout;" in h


def test_header_chunk_budget_matches_spec():
    """tests/qlayout.py takes the chunk budget from include/usk.h's text (226,240 bytes)."""
    import os
    import re
    h = open(os.path.join(os.path.dirname(__file__), "..", "include", "usk.h")).read()
    nums = {int(m.replace(",", "")) for m in re.findall(r"(\d{3},\d{3}) bytes", h)}
    assert qlayout.SMEM_CAP in nums, nums
