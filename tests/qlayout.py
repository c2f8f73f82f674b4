"""The query layout of include/usk.h (USK_LAYOUT_QUERY), written from the header's text -- test code
only, independent of paper_2506_17255_b200/csrc/packed.cu.

Per layer: units in chunks of 256 (32 key groups of 8); chunk k takes rows * maxN_k * 512 bytes
(maxN_k = the largest N_u of its units), chunks back to back from the layer's qbyte_begin, layers back
to back from 0.  Inside chunk k the 16-bit word at byte ((i * maxN_k + c) * 32 + g) * 16 + 2 v holds
cell (i, c) of unit 256 k + 8 g + v as rho16 = ((b << 1) | (b >> 15)) ^ 1 (b = bf16 bits), 0 where the
unit does not exist, c >= N_u or i >= M_u."""
import numpy as np

SMEM_CAP = 227 * 1024 - (64 + 16 * 16 * 16 + 1024)  # the header's shared-memory budget for a chunk


def chunk_width(ncols, rows):
    return 256 if rows * int(max(ncols)) * 512 <= SMEM_CAP else 128


def rho16(b):
    b = b.astype(np.uint32)
    return ((((b << 1) | (b >> 15)) & 0xFFFF) ^ 1).astype(np.uint16)


def unrho16(r):
    r = r.astype(np.uint32) ^ 1
    return (((r >> 1) | (r << 15)) & 0xFFFF).astype(np.uint16)


def layer_geometry(ncols, rows):
    """(chunk maxN list, chunk byte sizes, chunk width) of one layer from its per-unit N."""
    n = len(ncols)
    cw = chunk_width(ncols, rows)
    mx = [int(max(ncols[k:k + cw])) for k in range(0, n, cw)]
    return mx, [rows * m * 2 * cw for m in mx], cw


def model_offsets(ncols_per_layer, rows):
    off, out = 0, []
    for nc in ncols_per_layer:
        out.append(off)
        off += sum(layer_geometry(nc, rows)[1])
    return out, off


def pack_layer(cells_u16, offsets, ncols, nrows, rows):
    """Unit-major cells of ONE layer (offsets relative to the array) -> the layer's query bytes (uint16)."""
    mx, sizes, cw = layer_geometry(ncols, rows)
    out = np.zeros(sum(sizes) // 2, np.uint16)
    base = 0
    n = len(ncols)
    for k, m in enumerate(mx):
        words = out[base // 2:(base + sizes[k]) // 2].reshape(rows, m, cw)
        for u in range(k * cw, min(n, (k + 1) * cw)):
            t = u - k * cw
            N, M = int(ncols[u]), int(nrows[u])
            c = cells_u16[offsets[u]:offsets[u] + M * N].reshape(M, N)
            words[:M, :N, t] = rho16(c)
        base += sizes[k]
    return out


def unpack_layer(q_u16, offsets, ncols, nrows, rows):
    """Inverse of pack_layer: the unit-major cells of the layer (and whether the padding is 0)."""
    mx, sizes, cw = layer_geometry(ncols, rows)
    n = len(ncols)
    cells = np.zeros(int(offsets[n] - offsets[0]), np.uint16)
    pad_ok = True
    base = 0
    for k, m in enumerate(mx):
        words = q_u16[base // 2:(base + sizes[k]) // 2].reshape(rows, m, cw)
        seen = np.zeros(words.shape, bool)
        for u in range(k * cw, min(n, (k + 1) * cw)):
            t = u - k * cw
            N, M = int(ncols[u]), int(nrows[u])
            cells[offsets[u] - offsets[0]:offsets[u] - offsets[0] + M * N] = unrho16(words[:M, :N, t]).reshape(-1)
            seen[:M, :N, t] = True
        pad_ok &= bool((words[~seen] == 0).all())
        base += sizes[k]
    return cells, pad_ok


def unit_cells(q_u16, ncols, nrows, t, rows):
    """Unit-major cells (M_u * N_u, row-major) of unit t of a layer from the layer's query bytes."""
    mx, sizes, cw = layer_geometry(ncols, rows)
    k = t // cw
    base = sum(sizes[:k])
    words = q_u16[base // 2:(base + sizes[k]) // 2].reshape(rows, mx[k], cw)
    N, M = int(ncols[t]), int(nrows[t])
    return unrho16(words[:M, :N, t - k * cw]).reshape(-1)
