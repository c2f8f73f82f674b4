"""Multi-GPU orchestration of the sketch path (host side; torch.distributed for the plumbing).

SURVEY §8(e) / DESIGN.md "Multi-GPU":
  * Build: compression units are independent, so layers are sharded over ranks with
    no data-path collective; every rank computes the (deterministic) plan itself.  A one-time
    replication (one broadcast per layer region from its owner) gives every rank the full sketch
    for output-sharded inference.
  * Decode: each linear's output features are split into contiguous per-rank ranges; each rank
    runs usk_linear on its range and the fp32 y shards are all-gathered (NCCL on GPUs).
  * Output-row units (L31): each rank builds just the units of its own output rows
    (build_output_shard, usk_build_rows) and decodes that range -- disjoint sketch shards, no
    replication; the y shards are all-gathered as above.
  * Prefill: replicas (sequences sharded, sketch replicated) -- no collective.
"""
from __future__ import annotations


def output_shard(out_features: int, rank: int, world: int):
    """Contiguous output range [o0, o1) of `rank` (sizes differ by at most one row)."""
    return (out_features * rank) // world, (out_features * (rank + 1)) // world


def layer_owner(layer: int, world: int, layers_per_block: int = 7) -> int:
    """Owner rank of a layer for the sharded build: whole transformer blocks round-robin."""
    return (layer // layers_per_block) % world


def owned_layers(n_layers: int, rank: int, world: int, layers_per_block: int = 7):
    return [l for l in range(n_layers) if layer_owner(l, world, layers_per_block) == rank]


def build_output_shard(usk, plan, layer: int, w_full_or_rows, sketch, rank: int, world: int, rows_only=False,
                       stream=None):
    """Output-row units (L31): rank `rank` builds only the units of its output shard of
    `layer` (disjoint per-rank sketch regions: no replication step).  w_full_or_rows: the layer's
    full [out, in] weight, or (rows_only=True) just this rank's rows."""
    o0, o1 = output_shard(plan.layers[layer].out_features, rank, world)
    w_rows = w_full_or_rows if rows_only else w_full_or_rows[o0:o1]
    usk.build_rows(plan, layer, o0, o1, w_rows, sketch, stream=stream)
    return o0, o1


def replicate_sketch(sketch_bytes, layer_regions, world: int, group=None, layers_per_block: int = 7):
    """Broadcast every layer's byte region [b0, b1) of `sketch_bytes` (a uint8 tensor) from its
    owner so that all ranks hold the full sketch (one-time deployment step)."""
    import torch.distributed as dist
    for l, (b0, b1) in enumerate(layer_regions):
        if b1 > b0:
            dist.broadcast(sketch_bytes[b0:b1], src=layer_owner(l, world, layers_per_block), group=group)


def allgather_outputs(y_shard, y_full, group=None):
    """y_full[...] = concatenation over ranks of their y shards (equal-size shards use
    all_gather_into_tensor; ragged shards fall back to all_gather + copy).  Batch-1 decode only:
    y_shard and y_full are 1-D (one token)."""
    import torch
    import torch.distributed as dist
    if y_shard.dim() != 1 or y_full.dim() != 1:
        raise ValueError("allgather_outputs: 1-D (T = 1) shards only")
    world = dist.get_world_size(group)
    n = y_full.shape[-1]
    sizes = [output_shard(n, r, world) for r in range(world)]
    if all(b - a == sizes[0][1] - sizes[0][0] for a, b in sizes):
        dist.all_gather_into_tensor(y_full, y_shard.contiguous(), group=group)
        return y_full
    mx = max(b - a for a, b in sizes)  # pad the ragged shards to one size
    padded = torch.zeros(mx, dtype=y_shard.dtype, device=y_shard.device)
    padded[:y_shard.numel()] = y_shard
    parts = [torch.empty(mx, dtype=y_shard.dtype, device=y_shard.device) for _ in sizes]
    dist.all_gather(parts, padded, group=group)
    for (a, b), p in zip(sizes, parts):
        y_full[a:b] = p[:b - a]
    return y_full


# ---- one collective per grouped call: the linears of a group (q|k|v, o, gate|up,
#      down) write their y shards into ONE contiguous per-rank buffer, gathered by one all-gather
def group_shard_layout(out_features, rank: int, world: int):
    """Per layer of a group: (o0, o1, offset) of this rank's shard in the group's shard buffer, and
    the buffer length padded to the largest rank's (all_gather_into_tensor needs equal parts)."""
    lay, off = [], 0
    for o in out_features:
        o0, o1 = output_shard(o, rank, world)
        lay.append((o0, o1, off))
        off += o1 - o0
    pad = max(sum(output_shard(o, r, world)[1] - output_shard(o, r, world)[0] for o in out_features)
              for r in range(world))
    return lay, pad


def allgather_group(shard_buf, gathered, group=None):
    """gathered [world * len(shard_buf)] = every rank's shard buffer, rank-major (one collective)."""
    import torch.distributed as dist
    dist.all_gather_into_tensor(gathered, shard_buf, group=group)
    return gathered


def assemble_group(gathered, out_features, world: int):
    """Full y of each layer of a group from the rank-major gathered buffer (host-side check; a
    consumer of the decode reads the gathered buffer through the same layout)."""
    import torch
    pad = gathered.numel() // world
    parts = gathered.view(world, pad)
    ys = []
    for k, o in enumerate(out_features):
        pieces = []
        for r in range(world):
            lay, _ = group_shard_layout(out_features, r, world)
            o0, o1, off = lay[k]
            pieces.append(parts[r, off:off + (o1 - o0)])
        ys.append(torch.cat(pieces))
    return ys


# ---- fused y all-gather (usk_linear_batch_peers): the split-K reduce kernel of each rank
#      stores its rows straight into every rank's full y over NVLink and raises a flag; usk_peer_wait
#      completes the exchange.  The peer buffers come from torch symmetric memory (one rendezvous).
def peer_layout(group_out_features):
    """Byte layout of the symmetric buffer: every grouped call's full fp32 y (256-B aligned pieces, in
    call order), then one int32 signal array.  Returns (per-call offsets, signal offset, total bytes)."""
    offs, off = [], 0
    for outs in group_out_features:
        o = []
        for n_out in outs:
            o.append(off)
            off += (n_out * 4 + 255) // 256 * 256
        offs.append(o)
    return offs, off, off + 256


class PeerYBuffers:
    """Every grouped call's full-y buffers (fp32) and one signal array (int32[world]) in ONE symmetric-
    memory allocation, mapped on every rank; `peers(gi)` is the usk.Peers of grouped call gi."""

    def __init__(self, usk, group_out_features, device, group=None):
        import torch
        import torch.distributed as dist
        import torch.distributed._symmetric_memory as symm_mem
        self.world = dist.get_world_size(group)
        self.rank = dist.get_rank(group)
        offs, sig_off, total = peer_layout(group_out_features)
        self.buf = symm_mem.empty(total, dtype=torch.uint8, device=device)
        self.buf.zero_()
        self.handle = symm_mem.rendezvous(self.buf, group if group is not None else dist.group.WORLD)
        ptrs = [int(p) for p in self.handle.buffer_ptrs]
        self.epoch = torch.zeros(1, dtype=torch.int32, device=device)
        self.y = [[self.buf[a:a + n * 4].view(torch.float32) for a, n in zip(o, outs)]
                  for o, outs in zip(offs, group_out_features)]
        self.yflat = self.buf[:sig_off].view(torch.float32)  # every full y (256-B aligned pieces)
        self._peers = [usk.Peers(self.world, self.rank, [[p + a for a in o] for p in ptrs], [p + sig_off for p in ptrs],
                                 self.epoch) for o in offs]
        torch.cuda.synchronize(device)
        dist.barrier(group)  # every rank's signal array is zero before the first flag

    def peers(self, gi: int):
        return self._peers[gi]
