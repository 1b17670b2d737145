"""Oracle: box calculus and level metadata.  TEST INFRASTRUCTURE ONLY.

A box (patch) is P = [i_lo, i_hi], inclusive integer N-vectors.  Refinement and
coarsening per P:1026-1038: R(P) = [R lo, R (hi+1) - 1], C(P) = [floor(lo/R), floor(hi/R)].

Also here, as plain definitions of the metadata both sides must agree on bit-exactly:

* ghost maps: for every cell of grow(P, 2), where its value comes from (ordering rule of
  reading #15: velocity index outside the domain => PHYS; else a same-level patch (after the
  periodic wrap of configuration indices) => SIBLING; else the next coarser level => CF),
* Alg.7 ComputeSubPatches with the deterministic box difference of SPEC (split
  dim 0 first, low fragment before high), results sorted lexicographically,
* tag dilation and the C3 fixed-tile rule (reading #18).
"""
from __future__ import annotations

import itertools

import numpy as np

G = 2
INTERIOR, SIBLING, COARSE, PHYS = 0, 1, 2, 3


def box(lo, hi):
    return (tuple(int(x) for x in lo), tuple(int(x) for x in hi))


def is_empty(b):
    return any(l > h for l, h in zip(*b))


def size(b):
    return tuple(h - l + 1 for l, h in zip(*b))


def ncells(b):
    return 0 if is_empty(b) else int(np.prod(size(b)))


def refine(b, ratio):
    """R(P)."""
    lo, hi = b
    return box([l * r for l, r in zip(lo, ratio)], [(h + 1) * r - 1 for h, r in zip(hi, ratio)])


def coarsen(b, ratio):
    """C(P), P:1033 with floor division (negative indices behave uniformly)."""
    lo, hi = b
    return box([l // r for l, r in zip(lo, ratio)], [h // r for h, r in zip(hi, ratio)])


def grow(b, g):
    lo, hi = b
    gs = g if isinstance(g, (tuple, list)) else (g,) * len(lo)
    return box([l - x for l, x in zip(lo, gs)], [h + x for h, x in zip(hi, gs)])


def intersect(a, b):
    return box([max(x, y) for x, y in zip(a[0], b[0])], [min(x, y) for x, y in zip(a[1], b[1])])


def contains_cell(b, c):
    return all(l <= x <= h for l, x, h in zip(b[0], c, b[1]))


def contains_box(outer, inner):
    return all(ol <= il and ih <= oh for ol, il, ih, oh in zip(outer[0], inner[0], inner[1], outer[1]))


def restr(b, dims):
    """restr_j: drop the listed dims."""
    keep = [d for d in range(len(b[0])) if d not in set(dims)]
    return box([b[0][d] for d in keep], [b[1][d] for d in keep])


def repl(b, d, a, c):
    """repl_j(a, b)."""
    lo, hi = list(b[0]), list(b[1])
    lo[d], hi[d] = a, c
    return box(lo, hi)


def subtract(a, b):
    """a minus b as disjoint boxes: split dim 0 first, low fragment before high."""
    if is_empty(intersect(a, b)):
        return [a]
    out = []
    lo, hi = list(a[0]), list(a[1])
    for d in range(len(lo)):
        if lo[d] < b[0][d]:
            h2 = list(hi); h2[d] = b[0][d] - 1
            out.append(box(lo, h2))
            lo[d] = b[0][d]
        if hi[d] > b[1][d]:
            l2 = list(lo); l2[d] = b[1][d] + 1
            out.append(box(l2, hi))
            hi[d] = b[1][d]
    return out


def sort_boxes(bs):
    return sorted(bs, key=lambda b: (b[0], b[1]))


def cell_index(b, c):
    """Row-major linear index of cell c inside box b (last dim fastest)."""
    idx = 0
    for d in range(len(c)):
        idx = idx * (b[1][d] - b[0][d] + 1) + (c[d] - b[0][d])
    return idx


def cells_of(b):
    return itertools.product(*[range(l, h + 1) for l, h in zip(*b)])


# --------------------------------------------------------------------------- levels
class LevelMeta:
    """Boxes of one level in its own index space, with the ratio to level 0."""

    def __init__(self, domain0, ratio_to_0, boxes, periodic):
        self.ratio = tuple(int(r) for r in ratio_to_0)
        self.domain = refine(domain0, self.ratio)
        self.boxes = [box(*b) for b in boxes]
        self.periodic = tuple(bool(p) for p in periodic)
        self.ndim = len(self.ratio)

    def wrap(self, c):
        out = []
        for d, x in enumerate(c):
            if self.periodic[d]:
                lo, hi = self.domain[0][d], self.domain[1][d]
                n = hi - lo + 1
                x = lo + (x - lo) % n
            out.append(x)
        return tuple(out)

    def find(self, c):
        for p, b in enumerate(self.boxes):
            if contains_cell(b, c):
                return p
        return -1


def ghost_map(level, p, coarser=None):
    """Dense ghost map of patch p over grow(box, G), row-major.  Returns (kind, src_patch,
    src_cell) int arrays.  Encoding (shared with include/vlasov.h):
      INTERIOR: src_patch = p, src_cell = index in box p
      SIBLING : src_patch = q (may equal p across the periodic wrap), src_cell = index of the
                wrapped cell in box q
      COARSE  : src_patch = coarse patch whose box holds the coarse parent of the wrapped cell,
                src_cell = index of that parent in it
      PHYS    : src_patch = -1, src_cell = 2*(velocity dim number) + (0 low | 1 high), for the
                first velocity axis whose index lies outside the domain."""
    b = level.boxes[p]
    gb = grow(b, G)
    ncfg = level.ndim // 2
    n = ncells(gb)
    kind = np.zeros(n, np.int32)
    src_p = np.zeros(n, np.int32)
    src_c = np.zeros(n, np.int64)
    for t, c in enumerate(cells_of(gb)):
        if contains_cell(b, c):
            kind[t], src_p[t], src_c[t] = INTERIOR, p, cell_index(b, c)
            continue
        phys = -1
        for vd in range(ncfg, level.ndim):
            if c[vd] < level.domain[0][vd]:
                phys = 2 * (vd - ncfg)
                break
            if c[vd] > level.domain[1][vd]:
                phys = 2 * (vd - ncfg) + 1
                break
        if phys >= 0:
            kind[t], src_p[t], src_c[t] = PHYS, -1, phys
            continue
        w = level.wrap(c)
        q = level.find(w)
        if q >= 0:
            kind[t], src_p[t], src_c[t] = SIBLING, q, cell_index(level.boxes[q], w)
            continue
        if coarser is None:
            raise ValueError(f"ghost cell {c} of patch {p} has no source (level not covering)")
        rr = tuple(f // cr for f, cr in zip(level.ratio, coarser.ratio))
        cc = tuple(x // r for x, r in zip(w, rr))
        cq = coarser.find(cc)
        if cq < 0:
            raise ValueError(f"ghost cell {c} of patch {p}: coarse parent {cc} not on coarser level")
        kind[t], src_p[t], src_c[t] = COARSE, cq, cell_index(coarser.boxes[cq], cc)
    return kind, src_p, src_c


def properly_nested(fine, coarse):
    """Every fine box, coarsened, covered by the union of coarse boxes (Fig.1 caption)."""
    rr = tuple(f // c for f, c in zip(fine.ratio, coarse.ratio))
    for b in fine.boxes:
        for c in cells_of(coarsen(b, rr)):
            if coarse.find(c) < 0:
                return False
    return True


# --------------------------------------------------------------------------- Alg.7
def compute_sub_patches(p_in, level_index, hierarchy):
    """Alg.7 ComputeSubPatches.  ``hierarchy`` is a list of LevelMeta;
    ``p_in`` a box of level ``level_index``.  Finer boxes are coarsened to P_in's index space.
    Velocity (reduction) dims are the trailing half.  Returns sorted disjoint boxes."""
    lvl = hierarchy[level_index]
    ndim = lvl.ndim
    vdims = range(ndim // 2, ndim)
    S = [p_in]
    for fl in hierarchy[level_index + 1:]:
        rr = tuple(f // c for f, c in zip(fl.ratio, lvl.ratio))
        for fb in fl.boxes:
            P = coarsen(fb, rr)
            if is_empty(intersect(P, p_in)):
                continue
            P_ext = P
            for d in vdims:                                      # extend in reduction dims
                P_ext = repl(P_ext, d, p_in[0][d], p_in[1][d])
            newS = []
            for Ps in S:                                         # split by P_extend
                inter = intersect(Ps, P_ext)
                if is_empty(inter):
                    newS.append(Ps)
                    continue
                newS.append(inter)
                newS.extend(subtract(Ps, inter))
            S = []
            for Ps in newS:                                      # S <- S - P
                S.extend(subtract(Ps, P))
    return sort_boxes([s for s in S if not is_empty(s)])


# --------------------------------------------------------------------------- tags / tiles
def dilate_tags(tags, buffer, periodic):
    """Chebyshev dilation by ``buffer`` cells, periodic on the flagged axes, clipped otherwise."""
    t = np.asarray(tags, dtype=bool)
    if buffer <= 0:
        return t.copy()
    out = t.copy()
    for offs in itertools.product(range(-buffer, buffer + 1), repeat=t.ndim):
        shifted = t
        for ax, o in enumerate(offs):
            if o == 0:
                continue
            if periodic[ax]:
                shifted = np.roll(shifted, o, axis=ax)
            else:
                z = np.zeros_like(shifted)
                src = [slice(None)] * t.ndim
                dst = [slice(None)] * t.ndim
                if o > 0:
                    src[ax] = slice(0, t.shape[ax] - o); dst[ax] = slice(o, None)
                else:
                    src[ax] = slice(-o, None); dst[ax] = slice(0, t.shape[ax] + o)
                z[tuple(dst)] = shifted[tuple(src)]
                shifted = z
        out |= shifted
    return out


def tiles_from_tags(tags, ratio, tile):
    """C3 fixed-tile rule (reading #18): the level-0 domain refined by ``ratio`` is tiled by
    ``tile``-cell boxes; a tile exists iff its coarse footprint (tile/ratio cells per dim)
    holds a tagged cell.  Returns fine boxes sorted lexicographically."""
    t = np.asarray(tags, dtype=bool)
    foot = [tile // r for r in ratio]
    out = []
    for idx in itertools.product(*[range(t.shape[d] // foot[d]) for d in range(t.ndim)]):
        sl = tuple(slice(i * f, (i + 1) * f) for i, f in zip(idx, foot))
        if t[sl].any():
            out.append(box([i * tile for i in idx], [(i + 1) * tile - 1 for i in idx]))
    return sort_boxes(out)


# --------------------------------------------------------------------------- nesting (multi-level regrid)
def nesting_mask(level, buffer=1):
    """Cells of `level` (whole level domain) around which every cell within Chebyshev distance
    `buffer` lies in a patch of the level (configuration dims periodic; cells beyond the velocity
    domain count as covered): where a finer level may be placed so that it is properly nested
    (Fig.1 caption) with room for the coarse-fine stencils."""
    shape = size(level.domain)
    cov = np.zeros(shape, bool)
    for b in level.boxes:
        cov[tuple(slice(b[0][d], b[1][d] + 1) for d in range(level.ndim))] = True
    out = cov.copy()
    for offs in itertools.product(range(-buffer, buffer + 1), repeat=level.ndim):
        sh = cov
        for ax, o in enumerate(offs):
            if o == 0:
                continue
            if level.periodic[ax]:
                sh = np.roll(sh, -o, axis=ax)            # sh[c] = cov[c + o]
            else:
                z = np.ones_like(sh)                     # outside the velocity domain: covered
                src = [slice(None)] * level.ndim
                dst = [slice(None)] * level.ndim
                n = sh.shape[ax]
                if o > 0:
                    dst[ax] = slice(0, n - o); src[ax] = slice(o, n)
                else:
                    dst[ax] = slice(-o, n); src[ax] = slice(0, n + o)
                z[tuple(dst)] = sh[tuple(src)]
                sh = z
        out &= sh
    return out


def mask_to_boxes(mask, lo=(0, 0)):
    """Deterministic decomposition of a 2D boolean mask into disjoint boxes: maximal runs of True
    along the last dim in every row; a run continues its box while the next row has the identical
    run.  Boxes offset by `lo`, sorted lexicographically."""
    m = np.asarray(mask, bool)
    nx = m.shape[0]
    active = {}
    out = []

    def runs(row):
        r, j, n = [], 0, row.size
        while j < n:
            if row[j]:
                k = j
                while k + 1 < n and row[k + 1]:
                    k += 1
                r.append((j, k))
                j = k + 1
            else:
                j += 1
        return r
    for x in range(nx + 1):
        cur = runs(m[x]) if x < nx else []
        for run in sorted(list(active)):
            if run not in cur:
                out.append(box((lo[0] + active.pop(run), lo[1] + run[0]), (lo[0] + x - 1, lo[1] + run[1])))
        for run in cur:
            if run not in active:
                active[run] = x
    return sort_boxes(out)
