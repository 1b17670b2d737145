"""Pins of oracle/boxes.py: SPEC worked examples (cited), and cell-by-cell brute force on
seeded random hierarchies (sub-patch coverage, ghost-map sources, nesting)."""
import json
import os

import numpy as np
import pytest

from inputs.hierarchies import random_hierarchy
from oracle import boxes

EX = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "spec_box_examples.json")))


def B(b):
    return boxes.box(*b)


def test_spec_examples():
    for e in EX["refine"]:
        assert boxes.refine(B(e["box"]), e["R"]) == B(e["out"])
    for e in EX["coarsen"]:
        assert boxes.coarsen(B(e["box"]), e["R"]) == B(e["out"])
    for e in EX["restr"]:
        assert boxes.restr(B(e["box"]), e["dims"]) == B(e["out"])
    for e in EX["repl"]:
        assert boxes.repl(B(e["box"]), e["d"], e["a"], e["b"]) == B(e["out"])
    for e in EX["subtract"]:
        out = boxes.subtract(B(e["a"]), B(e["b"]))
        assert len(out) == e["nboxes"] and sum(boxes.ncells(b) for b in out) == e["ncells"]
    for e in EX["subpatches"]:
        coarse = boxes.LevelMeta(B(e["p_in"]), (1, 1), [B(e["p_in"])], (True, False))
        fine = boxes.LevelMeta(B(e["p_in"]), (1, 1), [B(e["finer_coarsened"])], (True, False))
        got = boxes.compute_sub_patches(B(e["p_in"]), 0, [coarse, fine])
        assert got == [B(b) for b in e["out"]]


def test_refine_coarsen_roundtrip_bruteforce():
    for R in (2, 3, 4):
        for lo in range(-8, 5):
            for hi in range(lo, 9):
                b = boxes.box((lo,), (hi,))
                assert boxes.coarsen(boxes.refine(b, (R,)), (R,)) == b


def test_subtract_partition_bruteforce():
    rng = np.random.default_rng(0)
    for _ in range(200):
        a = boxes.box(rng.integers(-3, 3, 2), rng.integers(3, 9, 2))
        lo = rng.integers(-5, 7, 2)
        b = boxes.box(lo, lo + rng.integers(0, 6, 2))
        parts = boxes.subtract(a, b)
        cells = [c for p in parts for c in boxes.cells_of(p)]
        assert len(cells) == len(set(cells))
        expect = {c for c in boxes.cells_of(a) if not boxes.contains_cell(b, c)}
        assert set(cells) == expect


def _meta(rat, lb):
    dom = boxes.box((0, 0), (lb[0][-1][1][0], lb[0][-1][1][1]))
    return [boxes.LevelMeta(dom, r, [B(b) for b in bl], (True, False)) for r, bl in zip(rat, lb)]


@pytest.mark.parametrize("seed", range(25))
def test_subpatches_tile_uncovered_cells(seed):
    # Alg.7 output, unioned with the coarsened finer footprints clipped to the patch, tiles the
    # patch exactly; every sub-patch spans the patch's whole v-range or is bounded by a finer
    # footprint (the extension step of P:1224).
    rat, lb = random_hierarchy(seed)
    H = _meta(rat, lb)
    for l, lvl in enumerate(H):
        for p_in in lvl.boxes:
            S = boxes.compute_sub_patches(p_in, l, H)
            cells = [c for s in S for c in boxes.cells_of(s)]
            assert len(cells) == len(set(cells)), "sub-patches overlap"
            covered = set()
            for fl in H[l + 1:]:
                rr = tuple(f // c for f, c in zip(fl.ratio, lvl.ratio))
                for fb in fl.boxes:
                    cb = boxes.intersect(boxes.coarsen(fb, rr), p_in)
                    if not boxes.is_empty(cb):
                        covered |= set(boxes.cells_of(cb))
            assert set(cells) == set(boxes.cells_of(p_in)) - covered
            assert S == boxes.sort_boxes(S)


@pytest.mark.parametrize("seed", range(25))
def test_ghost_map_sources_bruteforce(seed):
    rat, lb = random_hierarchy(seed)
    H = _meta(rat, lb)
    for l, lvl in enumerate(H):
        coarser = H[l - 1] if l else None
        for p, b in enumerate(lvl.boxes):
            kind, sp, sc = boxes.ghost_map(lvl, p, coarser)
            gb = boxes.grow(b, 2)
            assert kind.size == boxes.ncells(gb)
            for t, c in enumerate(boxes.cells_of(gb)):
                k = kind[t]
                if boxes.contains_cell(b, c):
                    assert k == boxes.INTERIOR and sp[t] == p
                    continue
                if c[1] < lvl.domain[0][1] or c[1] > lvl.domain[1][1]:
                    assert k == boxes.PHYS and sc[t] == (0 if c[1] < 0 else 1)
                    continue
                n = lvl.domain[1][0] + 1
                w = (c[0] % n, c[1])
                owners = [q for q, qb in enumerate(lvl.boxes) if boxes.contains_cell(qb, w)]
                if owners:
                    assert k == boxes.SIBLING and sp[t] == owners[0]
                    qb = lvl.boxes[owners[0]]
                    nv = qb[1][1] - qb[0][1] + 1
                    assert sc[t] == (w[0] - qb[0][0]) * nv + (w[1] - qb[0][1])
                else:
                    rr = tuple(f // cc for f, cc in zip(lvl.ratio, coarser.ratio))
                    par = (w[0] // rr[0], w[1] // rr[1])
                    assert k == boxes.COARSE and boxes.contains_cell(coarser.boxes[sp[t]], par)


@pytest.mark.parametrize("seed", range(10))
def test_random_hierarchies_are_nested(seed):
    rat, lb = random_hierarchy(seed)
    H = _meta(rat, lb)
    for l in range(1, len(H)):
        assert boxes.properly_nested(H[l], H[l - 1])


def test_nesting_counterexample():
    dom = boxes.box((0, 0), (7, 7))
    coarse = boxes.LevelMeta(dom, (1, 1), [boxes.box((0, 0), (3, 7))], (True, False))
    fine = boxes.LevelMeta(dom, (2, 2), [boxes.box((4, 0), (9, 3))], (True, False))
    assert not boxes.properly_nested(fine, coarse)


def test_tiles_and_dilation():
    t = np.zeros((16, 32), bool)
    t[5, 9] = True
    d = boxes.dilate_tags(t, 1, (True, False))
    assert d.sum() == 9 and d[4:7, 8:11].all()
    t2 = np.zeros((16, 32), bool)
    t2[0, 0] = True
    d2 = boxes.dilate_tags(t2, 1, (True, False))
    assert d2.sum() == 6 and d2[15, 0] and d2[1, 1] and not d2[0, 31]   # periodic x, clipped v
    tiles = boxes.tiles_from_tags(d, (4, 4), 32)                         # 8x8 coarse footprints
    assert tiles == [boxes.box((0, 32), (31, 63))]
