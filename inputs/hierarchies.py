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
