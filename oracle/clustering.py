"""Oracle: tag clustering into rectangular patches.  TEST INFRASTRUCTURE ONLY.

PAPER.md P:468-475: "cells that should be refined are tagged.  Tagged cells are grouped and
expanded minimally to form rectangular patches"; P:1495-1515 (Table tab:amr_param): per-level
largest_patch_size, smallest_patch_size, regrid_interval, tag_buffer.  The grouping algorithm is not
specified in the paper (SAMRAI's Berger-Rigoutsos is implied); reading #28
fixes this deterministic signature-based recursive bisection (SPEC.md "DESIGN DECISIONS"):

cluster(region R):
  1. B = bounding box of the tags in R; no tags -> nothing.
  2. if fill efficiency |tags in B| / |B| >= efficiency and every side of B <= largest: accept B.
  3. otherwise look for a cut of B (a cut at c along d splits into [lo_d, c-1] and [c, hi_d]; a
     cut is admissible if both parts have >= smallest_d cells along d), dims visited in order of
     decreasing length of B (ties: lower dim first):
       a. holes: c such that the signature (tag count per slice) of slice c-1 or slice c is zero;
          take the admissible one closest to the centre (ties: lower c);
       b. inflection: Laplacian L_i = s_{i-1} - 2 s_i + s_{i+1} (i = 1 .. n-2); cut c = i where
          L_{i-1} L_i < 0, largest |L_i - L_{i-1}| (ties: closest to the centre, then lower c);
       c. if some side of B exceeds largest, or no a/b cut exists in any dim: bisect the longest
          dim with an admissible cut at lo + n/2 (floor).
     with no admissible cut at all: accept B.
  4. recurse on the two parts (each re-trimmed to its tags).
Boxes larger than `largest` after step 3 are tiled into ceil(n/largest) near-equal pieces per dim.
Output sorted lexicographically.
"""
from __future__ import annotations

import numpy as np

from . import boxes


def _bbox(t, lo):
    idx = np.argwhere(t)
    if idx.size == 0:
        return None
    a = idx.min(axis=0)
    b = idx.max(axis=0)
    return [int(lo[d] + a[d]) for d in range(t.ndim)], [int(lo[d] + b[d]) for d in range(t.ndim)]


def _order(n):
    """dims by decreasing length, ties lower dim first"""
    return sorted(range(len(n)), key=lambda d: (-n[d], d))


def _find_cut(sub, n, smallest):
    """sub: tag array of the box B (local indices); returns (d, c_local) or None."""
    nd = sub.ndim
    order = _order(n)
    admissible = lambda d, c: c >= smallest[d] and n[d] - c >= smallest[d]
    for d in order:                                                   # a. holes
        axes = tuple(a for a in range(nd) if a != d)
        sig = sub.sum(axis=axes)
        cands = []
        for c in range(1, n[d]):
            if (sig[c - 1] == 0 or sig[c] == 0) and admissible(d, c):
                cands.append((abs(2 * c - n[d]), c))
        if cands:
            return d, min(cands)[1]
    for d in order:                                                   # b. inflection
        axes = tuple(a for a in range(nd) if a != d)
        sig = sub.sum(axis=axes).astype(np.int64)
        if n[d] < 3:
            continue
        lap = [int(sig[i - 1] - 2 * sig[i] + sig[i + 1]) for i in range(1, n[d] - 1)]   # lap[j] at i = j+1
        cands = []
        for j in range(1, len(lap)):
            if lap[j - 1] * lap[j] < 0:
                c = j + 1                                             # between slices j and j+1
                if admissible(d, c):
                    cands.append((-abs(lap[j] - lap[j - 1]), abs(2 * c - n[d]), c))
        if cands:
            return d, min(cands)[2]
    for d in order:                                                   # c. bisection
        c = n[d] // 2
        if admissible(d, c):
            return d, c
    return None


def _tile_large(b, largest):
    lo, hi = b
    nd = len(lo)
    ranges = []
    for d in range(nd):
        n = hi[d] - lo[d] + 1
        k = -(-n // largest[d])
        ranges.append([(lo[d] + (n * j) // k, lo[d] + (n * (j + 1)) // k - 1) for j in range(k)])
    out = []

    def rec(d, l, h):
        if d == nd:
            out.append(boxes.box(l, h))
            return
        for a, b2 in ranges[d]:
            rec(d + 1, l + [a], h + [b2])
    rec(0, [], [])
    return out


def cluster_tags(tags, smallest, largest, efficiency=0.7, lo=None):
    """Boxes (inclusive, level index space; `lo` = index of tags[0, ...]) covering every tag."""
    t = np.asarray(tags, dtype=bool)
    lo = tuple(lo) if lo is not None else (0,) * t.ndim
    out = []

    def rec(region_lo, sub):
        bb = _bbox(sub, region_lo)
        if bb is None:
            return
        blo, bhi = bb
        n = [bhi[d] - blo[d] + 1 for d in range(t.ndim)]
        S = sub[tuple(slice(blo[d] - region_lo[d], bhi[d] - region_lo[d] + 1) for d in range(t.ndim))]
        eff = S.sum() / float(np.prod(n))
        too_big = any(n[d] > largest[d] for d in range(t.ndim))
        if eff >= efficiency and not too_big:
            out.append(boxes.box(blo, bhi))
            return
        cut = _find_cut(S, n, smallest)
        if cut is None:
            out.extend(_tile_large(boxes.box(blo, bhi), largest) if too_big else [boxes.box(blo, bhi)])
            return
        d, c = cut
        left = tuple(slice(0, c) if a == d else slice(None) for a in range(t.ndim))
        right = tuple(slice(c, None) if a == d else slice(None) for a in range(t.ndim))
        rlo = list(blo)
        rlo[d] = blo[d] + c
        rec(list(blo), S[left])
        rec(rlo, S[right])

    rec(list(lo), t)
    return boxes.sort_boxes(out)
