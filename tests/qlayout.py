"""The query layout of include/usk.h (USK_LAYOUT_QUERY), written from the header's text -- test code
only, independent of paper_2506_17255_b200/csrc/packed.cu.

Per layer: key groups (units 8g..8g+7) in query order -- by the class of their units, stable (the
identity when every group has one class); query position q is unit 8 * order[q // 8] + q % 8.
Chunks cover consecutive query positions: CW_k positions (256 when M_k * maxN_k * 512 <= 226240
bytes, else 128, else 64), cut short at the layer end and, with several classes, at the next
class boundary; a one-class layer takes one CW from its largest M_u and N_u.  Chunk k takes
M_k * maxN_k * 2 * CW_k bytes; its 16-bit word at byte ((i * maxN_k + c) * CW_k + s) * 2 holds cell
(i, c) of the unit at query position q0_k + s as rho16 = ((b << 1) | (b >> 15)) ^ 1, 0 elsewhere."""
import numpy as np

SMEM_CAP = 226240  # the header's shared-memory budget for a chunk (bytes)


def chunk_width(ncols, rows):
    """One-class layer: the width from its widest units (rows = its largest M_u)."""
    m = int(max(ncols))
    for cw in (256, 128, 64):
        if rows * m * 2 * cw <= SMEM_CAP:
            return cw
    raise ValueError("no chunk width fits")


def rho16(b):
    b = b.astype(np.uint32)
    return ((((b << 1) | (b >> 15)) & 0xFFFF) ^ 1).astype(np.uint16)


def unrho16(r):
    r = r.astype(np.uint32) ^ 1
    return (((r >> 1) | (r << 15)) & 0xFFFF).astype(np.uint16)


def query_order(n_units, cls=None):
    """Group order of a layer: stable sort of the key groups by the class of their first unit."""
    G = n_units // 8
    if cls is None or len(set(int(c) for c in np.asarray(cls)[::8])) <= 1:
        return list(range(G))
    return sorted(range(G), key=lambda g: int(cls[8 * g]))


def chunks(ncols, nrows, rows, cls=None):
    """[(q0, n, cw, maxN, M)] of one layer and its group order, from per-unit N, M and classes."""
    n_units = len(ncols)
    order = query_order(n_units, cls)
    unit = lambda q: 8 * order[q // 8] + q % 8  # noqa: E731
    nr = np.full(n_units, rows) if nrows is None else np.asarray(nrows)
    multi = order != list(range(n_units // 8))
    out = []
    q = 0
    if not multi:
        cw = chunk_width(ncols, int(nr.max()))
    while q < n_units:
        end = n_units
        if multi:
            c0 = int(cls[unit(q)])
            end = q
            while end < n_units and int(cls[unit(end)]) == c0:
                end += 8
            for w in (256, 128, 64):
                e = min(q + w, end)
                mx = max(int(ncols[unit(t)]) for t in range(q, e))
                mr = max(int(nr[unit(t)]) for t in range(q, e))
                if mr * mx * 2 * w <= SMEM_CAP:
                    cw = w
                    break
            else:
                raise ValueError("no chunk width fits")
        e = min(q + cw, end)
        mx = max(int(ncols[unit(t)]) for t in range(q, e))
        mr = max(int(nr[unit(t)]) for t in range(q, e))
        out.append((q, e - q, cw, mx, mr))
        q = e
    return out, order


def layer_geometry(ncols, rows, nrows=None, cls=None):
    """(chunk maxN list, chunk byte sizes, width of the first chunk) of one layer."""
    ch, _ = chunks(ncols, nrows, rows, cls)
    return [c[3] for c in ch], [c[4] * c[3] * 2 * c[2] for c in ch], ch[0][2]


def model_offsets(ncols_per_layer, rows, nrows_per_layer=None, cls_per_layer=None):
    off, out = 0, []
    for k, nc in enumerate(ncols_per_layer):
        out.append(off)
        nr = None if nrows_per_layer is None else nrows_per_layer[k]
        cl = None if cls_per_layer is None else cls_per_layer[k]
        off += sum(layer_geometry(nc, rows, nr, cl)[1])
    return out, off


def _slices(q_u16, ncols, nrows, rows, cls):
    ch, order = chunks(ncols, nrows, rows, cls)
    base = 0
    for (q0, n, cw, mx, mr) in ch:
        words = q_u16[base // 2:(base + mr * mx * 2 * cw) // 2].reshape(mr, mx, cw)
        yield words, [(s, 8 * order[(q0 + s) // 8] + (q0 + s) % 8) for s in range(n)]
        base += mr * mx * 2 * cw


def pack_layer(cells_u16, offsets, ncols, nrows, rows, cls=None):
    """Unit-major cells of ONE layer (offsets relative to the array) -> the layer's query bytes (uint16)."""
    mx, sizes, _ = layer_geometry(ncols, rows, nrows, cls)
    out = np.zeros(sum(sizes) // 2, np.uint16)
    for words, slots in _slices(out, ncols, nrows, rows, cls):
        for s, u in slots:
            N, M = int(ncols[u]), int(nrows[u])
            c = cells_u16[offsets[u]:offsets[u] + M * N].reshape(M, N)
            words[:M, :N, s] = rho16(c)
    return out


def unpack_layer(q_u16, offsets, ncols, nrows, rows, cls=None):
    """Inverse of pack_layer: the unit-major cells of the layer (and whether the padding is 0)."""
    n = len(ncols)
    cells = np.zeros(int(offsets[n] - offsets[0]), np.uint16)
    pad_ok = True
    for words, slots in _slices(q_u16, ncols, nrows, rows, cls):
        seen = np.zeros(words.shape, bool)
        for s, u in slots:
            N, M = int(ncols[u]), int(nrows[u])
            cells[offsets[u] - offsets[0]:offsets[u] - offsets[0] + M * N] = unrho16(words[:M, :N, s]).reshape(-1)
            seen[:M, :N, s] = True
        pad_ok &= bool((words[~seen] == 0).all())
    return cells, pad_ok


def unit_cells(q_u16, ncols, nrows, t, rows, cls=None):
    """Unit-major cells (M_u * N_u, row-major) of unit t of a layer from the layer's query bytes."""
    for words, slots in _slices(q_u16, ncols, nrows, rows, cls):
        for s, u in slots:
            if u == t:
                N, M = int(ncols[t]), int(nrows[t])
                return unrho16(words[:M, :N, s]).reshape(-1)
    raise KeyError(t)
