"""Seeded random box hierarchies for metadata / reduction parity tests (inputs only: integer
box lists, no method arithmetic).

A hierarchy is (ratios_to_level0, level_boxes): level 0 tiles the whole 1D+1V domain with
patches; level l+1 boxes are aligned unions of refined level-l cells, disjoint, and nested one
coarse cell inside the level-l union (so every coarse stencil of a CF ghost lies in level l).
"""
from __future__ import annotations

import numpy as np


def _tile(nx, nv, px, pv):
    out = []
    for x0 in range(0, nx, px):
        for v0 in range(0, nv, pv):
            out.append(((x0, v0), (min(x0 + px, nx) - 1, min(v0 + pv, nv) - 1)))
    return out


def _covered(boxes, shape):
    m = np.zeros(shape, bool)
    for (lo, hi) in boxes:
        m[lo[0]:hi[0] + 1, lo[1]:hi[1] + 1] = True
    return m


def random_hierarchy(seed, nx0=16, nv0=32, nlevels=None, ratios=(2, 4), max_boxes=4):
    """Random properly nested hierarchy on an nx0 x nv0 level-0 domain.
    Returns (ratios_to_level0 list, level_boxes list)."""
    rng = np.random.default_rng(seed)
    nlevels = nlevels or int(rng.integers(2, 4))
    px = int(rng.choice([4, 8, nx0]))
    pv = int(rng.choice([8, 16, nv0]))
    levels = [_tile(nx0, nv0, px, pv)]
    rat = [(1, 1)]
    for l in range(1, nlevels):
        r = (int(rng.choice(ratios)), int(rng.choice(ratios)))
        cur = rat[-1]
        nxl, nvl = nx0 * cur[0], nv0 * cur[1]
        cov = _covered(levels[-1], (nxl, nvl))
        # shrink the parent coverage by one coarse cell (nesting buffer): x periodic, and cells
        # beyond the v-domain count as covered (fine patches may touch the v boundary)
        pad = np.pad(cov, ((0, 0), (1, 1)), constant_values=True)
        inner = np.ones_like(cov)
        for dx in (-1, 0, 1):
            for dv in (-1, 0, 1):
                inner &= np.roll(pad, dx, axis=0)[:, 1 + dv: 1 + dv + nvl]
        boxes = []
        taken = np.zeros_like(cov)
        for _ in range(int(rng.integers(1, max_boxes + 1))):
            for _try in range(20):
                w = int(rng.integers(2, max(3, nxl // 3)))
                h = int(rng.integers(2, max(3, nvl // 3)))
                x0 = int(rng.integers(0, nxl - w + 1))
                v0 = int(rng.integers(0, nvl - h + 1))
                sl = (slice(x0, x0 + w), slice(v0, v0 + h))
                if inner[sl].all() and not taken[sl].any():
                    taken[sl] = True
                    boxes.append(((x0 * r[0], v0 * r[1]), ((x0 + w) * r[0] - 1, (v0 + h) * r[1] - 1)))
                    break
        if not boxes:
            break
        levels.append(sorted(boxes))
        rat.append((cur[0] * r[0], cur[1] * r[1]))
    return rat, levels


def random_hierarchy_4d(seed, n0=(8, 8, 8, 8), patch0=(8, 8, 4, 8), nlevels=2, ratios=(2,), max_boxes=2):
    """Random properly nested 2D+2V hierarchy (N3): level 0 tiles the (x, y, v_x, v_y) domain with
    patch0 boxes; every finer box is the refinement (ratio per dim from `ratios`) of a box of
    cells of the coarser level lying one coarse cell inside its union (x, y periodic; cells
    beyond the velocity domain count as covered, so fine boxes may touch it).  Returns
    (ratios_to_level0, level_boxes)."""
    import itertools
    rng = np.random.default_rng(seed)
    lv0 = []
    for lo in itertools.product(*[range(0, n0[d], patch0[d]) for d in range(4)]):
        lv0.append((tuple(lo), tuple(min(lo[d] + patch0[d], n0[d]) - 1 for d in range(4))))
    levels, rat = [sorted(lv0)], [(1, 1, 1, 1)]
    for _ in range(1, nlevels):
        r = tuple(int(rng.choice(ratios)) for _ in range(4))
        cur = rat[-1]
        nl = tuple(n0[d] * cur[d] for d in range(4))
        cov = np.zeros(nl, bool)
        for lo, hi in levels[-1]:
            cov[tuple(slice(lo[d], hi[d] + 1) for d in range(4))] = True
        pad = np.pad(cov, ((0, 0), (0, 0), (1, 1), (1, 1)), constant_values=True)
        inner = np.ones_like(cov)
        for off in itertools.product((-1, 0, 1), repeat=4):
            sh = np.roll(np.roll(pad, off[0], axis=0), off[1], axis=1)
            inner &= sh[:, :, 1 + off[2]: 1 + off[2] + nl[2], 1 + off[3]: 1 + off[3] + nl[3]]
        boxes, taken = [], np.zeros_like(cov)
        for _b in range(int(rng.integers(1, max_boxes + 1))):
            for _try in range(40):
                w = [int(rng.integers(2, max(3, nl[d] // 2 + 1))) for d in range(4)]
                lo = [int(rng.integers(0, nl[d] - w[d] + 1)) for d in range(4)]
                # velocity extent: touch the boundary or stay >= 2 coarse cells away from it
                ok = all(lo[d] == 0 or lo[d] >= 2 for d in (2, 3)) and \
                    all(lo[d] + w[d] == nl[d] or lo[d] + w[d] <= nl[d] - 2 for d in (2, 3))
                sl = tuple(slice(lo[d], lo[d] + w[d]) for d in range(4))
                if ok and inner[sl].all() and not taken[sl].any():
                    taken[sl] = True
                    boxes.append((tuple(lo[d] * r[d] for d in range(4)),
                                  tuple((lo[d] + w[d]) * r[d] - 1 for d in range(4))))
                    break
        if not boxes:
            break
        levels.append(sorted(boxes))
        rat.append(tuple(cur[d] * r[d] for d in range(4)))
    return rat, levels
