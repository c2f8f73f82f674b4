"""Multi-process (gloo, world size 2, CPU) tests of the multi-GPU host logic: layer-sharded build
+ sketch replication, and output-sharded decode + all-gather.  The per-rank compute is done by the
CPU oracle here (no GPU); the assembled results must equal the single-process oracle results
bit for bit (the GPU path is checked against the oracle elsewhere)."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import synth


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, shapes, q):
    import oracle
    from paper_2506_17255_b200 import dist as udist
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        opl = oracle.plan(shapes, 2.0, M=3, dtype=oracle.BF16, seed=11)
        Ws = [synth.weights_bf16(o, i, 50 + l) for l, (o, i) in enumerate(shapes)]
        # layer-sharded build: only owned layers are written locally
        sk = np.zeros(opl.total_cells, np.uint16)
        for l in udist.owned_layers(len(shapes), rank, world, layers_per_block=2):
            oracle.build_layer(opl, l, Ws[l], sk)
        t = torch.from_numpy(sk.view(np.uint8).copy())
        regions = []
        for l in range(len(shapes)):
            u0, u1 = opl.layer_units(l)
            regions.append((int(opl.offsets[u0]) * 2, int(opl.offsets[u1]) * 2))
        udist.replicate_sketch(t, regions, world, layers_per_block=2)
        full = t.numpy().view(np.uint16)
        # output-sharded decode of every layer, then all-gather
        ys = []
        for l, (o, i) in enumerate(shapes):
            x = synth.vector(i, seed=l)[0].astype(np.float64)
            o0, o1 = udist.output_shard(o, rank, world)
            y_shard = torch.from_numpy(oracle.linear_rows(opl, full, l, x, o0, o1)[0])
            y = torch.zeros(o, dtype=torch.float64)
            udist.allgather_outputs(y_shard, y)
            ys.append(y.numpy())
        if rank == 0:
            q.put((full.copy(), ys))
    except Exception as e:  # surface worker failures instead of a queue timeout
        q.put(("error", repr(e)))
        raise
    finally:
        dist.destroy_process_group()


def test_sharded_build_and_decode_gloo(orc):
    shapes = [(64, 96), (48, 64), (70, 96), (33, 64)]   # odd out sizes -> ragged shards
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, shapes, q)) for r in range(world)]
    for p in procs:
        p.start()
    full, ys = q.get(timeout=120)
    assert not isinstance(full, str), ys
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    opl = orc.plan(shapes, 2.0, M=3, dtype=orc.BF16, seed=11)
    Ws = [synth.weights_bf16(o, i, 50 + l) for l, (o, i) in enumerate(shapes)]
    ref = orc.build_model(opl, Ws)
    assert np.array_equal(full, ref)
    for l, (o, i) in enumerate(shapes):
        x = synth.vector(i, seed=l)[0].astype(np.float64)
        assert np.array_equal(ys[l], orc.linear_rows(opl, ref, l, x)[0])


def test_shard_helpers():
    from paper_2506_17255_b200 import dist as udist
    for out in (1, 7, 512, 2048, 14336):
        for world in (1, 2, 3, 8):
            r = [udist.output_shard(out, k, world) for k in range(world)]
            assert r[0][0] == 0 and r[-1][1] == out
            assert all(r[k][1] == r[k + 1][0] for k in range(world - 1))
            assert max(b - a for a, b in r) - min(b - a for a, b in r) <= 1
    owned = [udist.owned_layers(224, r, 8) for r in range(8)]
    assert sorted(l for o in owned for l in o) == list(range(224))
    assert all(len(o) == 28 for o in owned)


def _worker_outrow(rank, world, port, shapes, q):
    """Output-row units (L31): every rank builds only the units of its own output rows
    (disjoint sketch regions, no replication) and decodes that range; y shards are all-gathered."""
    import oracle
    from paper_2506_17255_b200 import dist as udist
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        opl = oracle.plan(shapes, 2.0, M=3, dtype=oracle.BF16, gran=oracle.GRAN_OUTROW, seed=13)
        ys, owned_cells = [], []
        sk = np.full(opl.total_cells, 0xABCD, np.uint16)      # cells of other ranks' rows stay garbage
        for l, (o, i) in enumerate(shapes):
            o0, o1 = udist.output_shard(o, rank, world)
            W = synth.weights_bf16(o, i, 60 + l)
            oracle.build_layer(opl, l, W, sk, t_begin=o0, t_end=o1)   # units = rows [o0, o1)
            u0, _ = opl.layer_units(l)
            owned_cells.append((int(opl.offsets[u0 + o0]), int(opl.offsets[u0 + o1])))
            x = synth.vector(i, seed=l)[0].astype(np.float64)
            y_shard = torch.from_numpy(oracle.linear_rows(opl, sk, l, x, o0, o1)[0])
            y = torch.zeros(o, dtype=torch.float64)
            udist.allgather_outputs(y_shard, y)
            ys.append(y.numpy())
        parts = [sk[a:b].copy() for a, b in owned_cells]
        if rank == 0:
            q.put(("ys", ys))
        q.put((rank, owned_cells, parts))
    except Exception as e:
        q.put(("error", repr(e)))
        raise
    finally:
        dist.destroy_process_group()


def test_outrow_disjoint_shards_gloo(orc):
    shapes = [(64, 96), (47, 64), (70, 32)]
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker_outrow, args=(r, world, port, shapes, q)) for r in range(world)]
    for p in procs:
        p.start()
    got = [q.get(timeout=120) for _ in range(world + 1)]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    assert not any(g[0] == "error" for g in got), got
    opl = orc.plan(shapes, 2.0, M=3, dtype=orc.BF16, gran=orc.GRAN_OUTROW, seed=13)
    ref = orc.build_model(opl, [synth.weights_bf16(o, i, 60 + l) for l, (o, i) in enumerate(shapes)])
    ys = next(g[1] for g in got if g[0] == "ys")
    covered = np.zeros(opl.total_cells, bool)
    for g in got:
        if g[0] in ("ys", "error"):
            continue
        for (a, b), part in zip(g[1], g[2]):
            np.testing.assert_array_equal(part, ref[a:b])       # each rank's own cells = the full build's
            assert not covered[a:b].any()                       # disjoint
            covered[a:b] = True
    assert covered.all()                                        # the shards tile the whole sketch
    for l, (o, i) in enumerate(shapes):
        x = synth.vector(i, seed=l)[0].astype(np.float64)
        np.testing.assert_array_equal(ys[l], orc.linear_rows(opl, ref, l, x)[0])


def test_peer_layout_host_logic():
    """dist.peer_layout (the symmetric buffer behind usk_linear_batch_peers): every grouped call's
    full y has its own 256-B aligned, non-overlapping piece in call order, and the signal array
    follows them."""
    from paper_2506_17255_b200 import dist as udist
    groups = [[3072, 512, 512], [2048], [8192, 8192], [2048]]
    offs, sig_off, total = udist.peer_layout(groups)
    spans = [(a, a + n * 4) for o, outs in zip(offs, groups) for a, n in zip(o, outs)]
    for (a0, a1), (b0, b1) in zip(spans, spans[1:]):
        assert a0 % 256 == 0 and a1 <= b0
    assert spans[-1][1] <= sig_off and sig_off % 256 == 0 and total >= sig_off + 4 * 8
