"""Pins of the oracle's tag clustering (oracle/clustering.py, reading #28): the SPEC.md examples,
and on seeded random tag fields the properties the paper's statement fixes (every
tagged cell lies in a patch; rectangular, disjoint patches) plus the AMR parameters' limits
(smallest / largest patch size) and the fill-efficiency stopping rule."""
import numpy as np
import pytest

from oracle import boxes, clustering


def _check(tags, bx, smallest, largest, eff, lo=(0, 0)):
    t = np.asarray(tags, bool)
    cov = np.zeros(t.shape, np.int32)
    for (a, b) in bx:
        sl = tuple(slice(a[d] - lo[d], b[d] - lo[d] + 1) for d in range(t.ndim))
        cov[sl] += 1
        n = [b[d] - a[d] + 1 for d in range(t.ndim)]
        assert all(n[d] <= largest[d] for d in range(t.ndim)), (a, b)
        # efficient, or not splittable any more (no admissible cut: every side < 2 smallest), or
        # a piece of the largest-size tiling
        e = t[sl].sum() / np.prod(n)
        assert e >= eff or all(n[d] < 2 * smallest[d] for d in range(t.ndim)) or \
            any(n[d] >= largest[d] // 2 for d in range(t.ndim)), (a, b, e)
    assert cov.max() <= 1                                   # disjoint
    assert np.all(cov[t] == 1)                              # every tag covered


def test_spec_examples():
    t = np.zeros((16, 16), bool)
    t[4:8, 4:10] = True
    assert clustering.cluster_tags(t, (2, 2), (16, 16)) == [((4, 4), (7, 9))]
    assert clustering.cluster_tags(np.zeros((8, 8), bool), (2, 2), (8, 8)) == []
    t = np.zeros((32, 32), bool)
    t[2:5, 3:6] = True
    t[25:30, 20:28] = True
    bx = clustering.cluster_tags(t, (2, 2), (32, 32))
    assert bx == [((2, 3), (4, 5)), ((25, 20), (29, 27))]


def test_largest_size_split_and_offset():
    t = np.ones((40, 10), bool)
    bx = clustering.cluster_tags(t, (4, 4), (16, 16), lo=(100, 7))
    # no hole, no inflection: bisection until every side <= largest
    assert bx == [((100, 7), (109, 16)), ((110, 7), (119, 16)), ((120, 7), (129, 16)), ((130, 7), (139, 16))]


@pytest.mark.parametrize("seed", range(25))
def test_random_fields_properties(seed):
    rng = np.random.default_rng(seed)
    shape = (int(rng.integers(8, 64)), int(rng.integers(8, 64)))
    t = np.zeros(shape, bool)
    for _ in range(int(rng.integers(1, 6))):                 # a few blobs plus noise
        c = [int(rng.integers(0, s)) for s in shape]
        r = [int(rng.integers(1, 8)) for _ in shape]
        t[max(0, c[0] - r[0]):c[0] + r[0], max(0, c[1] - r[1]):c[1] + r[1]] = True
    t |= rng.random(shape) < 0.01
    smallest = (int(rng.choice([2, 4])), int(rng.choice([2, 4])))
    largest = (int(rng.choice([16, 32, 64])), int(rng.choice([16, 32, 64])))
    eff = float(rng.choice([0.5, 0.7, 0.9]))
    bx = clustering.cluster_tags(t, smallest, largest, eff)
    _check(t, bx, smallest, largest, eff)
    assert bx == clustering.cluster_tags(t, smallest, largest, eff)       # deterministic


def test_efficiency_one_gives_exact_cover_of_rectangles():
    t = np.zeros((20, 20), bool)
    t[0:3, 0:20] = True
    t[10:20, 5:7] = True
    bx = clustering.cluster_tags(t, (1, 1), (64, 64), 1.0)
    assert sum(boxes.ncells(b) for b in bx) == t.sum()


# ---- the C-ABI clustering (host code of libvlasov) is bit-exact with the oracle
from paper_1204_3853_b200 import api  # noqa: E402


@pytest.mark.parametrize("seed", range(40))
def test_cabi_cluster_bitexact_vs_oracle(seed):
    rng = np.random.default_rng(1000 + seed)
    shape = (int(rng.integers(4, 80)), int(rng.integers(4, 80)))
    t = np.zeros(shape, bool)
    for _ in range(int(rng.integers(0, 6))):
        c = [int(rng.integers(0, s)) for s in shape]
        r = [int(rng.integers(1, 10)) for _ in shape]
        t[max(0, c[0] - r[0]):c[0] + r[0], max(0, c[1] - r[1]):c[1] + r[1]] = True
    t |= rng.random(shape) < float(rng.choice([0.0, 0.005, 0.03]))
    smallest = (int(rng.choice([1, 2, 4, 8])), int(rng.choice([1, 2, 4, 8])))
    largest = (int(rng.choice([8, 16, 32, 128])), int(rng.choice([8, 16, 32, 128])))
    largest = (max(largest[0], smallest[0]), max(largest[1], smallest[1]))
    eff = float(rng.choice([0.3, 0.7, 0.85, 1.0]))
    lo = (int(rng.integers(0, 50)), int(rng.integers(0, 50)))
    exp = clustering.cluster_tags(t, smallest, largest, eff, lo=lo)
    got = api.vlasov_cluster_tags(t.astype(np.uint8), smallest, largest, eff, lo=lo)
    assert got == [(tuple(b[0]), tuple(b[1])) for b in exp]


def test_cabi_cluster_c3_tags_amr_params():
    """C3 initial tags (paper's delta1+delta2 criterion, reading #18) clustered with the paper's
    AMR1 / AMR2 level-0 parameters after the tag buffer: C ABI == oracle."""
    import inputs
    from oracle import amr
    import amr_drivers as drv
    w = inputs.get("C3")
    H = drv.hierarchy(w, [inputs.level0_boxes(w)], [(1, 1)])
    data = H.new_data()
    for p, b in enumerate(H.levels[0].boxes):
        data[0][p][2:-2, 2:-2] = inputs.initial_cell_averages(w, (1, 1), b)
    amr.fill_ghosts(H, data, drv.zero_E(H))
    raw = amr.level0_tags(H, data, w.amr["tol"])
    for smallest, largest, buf in (((4, 4), (32, 32), 1), ((8, 8), (16, 32), 4)):
        t = boxes.dilate_tags(raw, buf, (True, False))
        exp = clustering.cluster_tags(t, smallest, largest, 0.7)
        got = api.vlasov_cluster_tags(t.astype(np.uint8), smallest, largest, 0.7)
        assert got == [(tuple(b[0]), tuple(b[1])) for b in exp]
        assert 0 < len(got) < 200


def test_mask_to_boxes_exact_cover():
    rng = np.random.default_rng(5)
    for _ in range(20):
        m = rng.random((int(rng.integers(1, 20)), int(rng.integers(1, 20)))) < 0.6
        bx = boxes.mask_to_boxes(m, (3, -2))
        cov = np.zeros(m.shape, int)
        for (a, b) in bx:
            cov[a[0] - 3: b[0] - 3 + 1, a[1] + 2: b[1] + 2 + 1] += 1
        assert np.array_equal(cov, m.astype(int))


@pytest.mark.parametrize("seed", range(20))
def test_cabi_regrid_boxes_bitexact_vs_oracle(seed):
    """Next-level boxes from tags under the proper-nesting constraint (reading #28): C ABI == oracle,
    and the result is properly nested (Fig.1 caption) with a one-cell buffer."""
    import inputs
    from inputs.hierarchies import random_hierarchy
    from oracle import amr
    rng = np.random.default_rng(2000 + seed)
    rat, lb = random_hierarchy(seed)
    w = inputs.scaled(inputs.get("C3"), (16, 32), (8, 8))
    levels = []
    for r, bl in zip(rat, lb):
        levels.append(api.Level(2, w.ncells, w.lower, inputs.spacing(w), r, bl, coarser=levels[-1] if levels else None))
    dom = boxes.box((0, 0), (15, 31))
    metas = [boxes.LevelMeta(dom, r, [boxes.box(*b) for b in bl], (True, False)) for r, bl in zip(rat, lb)]
    k = len(levels) - 1
    shape = boxes.size(metas[k].domain)
    t = rng.random(shape) < 0.05
    ratio = (int(rng.choice([2, 4])), int(rng.choice([2, 4])))
    sm, lg, eff = (4, 4), (32, 64), float(rng.choice([0.5, 0.7]))
    exp = amr.new_level_boxes(metas[k], t, ratio, sm, lg, eff)
    got = api.vlasov_regrid_boxes(levels[k].h, t.astype(np.uint8), ratio, sm, lg, eff)
    assert got == [(tuple(b[0]), tuple(b[1])) for b in exp]
    if exp:
        fine = boxes.LevelMeta(dom, tuple(a * b for a, b in zip(rat[k], ratio)), exp, (True, False))
        assert boxes.properly_nested(fine, metas[k])


def test_four_level_amr3_hierarchy_invariants():
    """The oracle's multi-level regrid with the paper's four-level ratios [2,4], [4,2], [2,2]
     and the AMR3 parameters (smallest (8,8); largest level_1 (32,128),
    level_2 (128,256), the finest specified value for level 3; tag buffer 8) on a C3-shaped
    16x32 base: four levels, every fine box a union of refined coarser cells, within the patch-size
    limits, pairwise disjoint, and properly nested in the next coarser level."""
    import sys
    import os
    sys.path.insert(0, os.path.dirname(__file__))
    import amr_drivers as drv
    import inputs
    w = inputs.scaled(inputs.get("C3"), (16, 32), (8, 8))
    ratios = [(2, 4), (4, 2), (2, 2)]
    smallest, largest = [(8, 8)] * 3, [(32, 128), (128, 256), (128, 256)]
    H = drv.hierarchy(w, [inputs.level0_boxes(w)], [(1, 1)])
    data = H.new_data()
    for p, b in enumerate(H.levels[0].boxes):
        data[0][p][2:-2, 2:-2] = inputs.initial_cell_averages(w, (1, 1), b)
    E_bc = drv.start(H, data)
    _, _, nbs = drv.regrid_multilevel(H, data, E_bc, 0.005, [8, 8, 8], ratios, smallest, largest, 0.7)
    assert len(nbs) == 3 and len(H.levels) == 4
    for k, nb in enumerate(nbs):
        r = ratios[k]
        dom = [w.ncells[d] * H.levels[k + 1].ratio[d] for d in range(2)]
        coarse = H.levels[k].boxes
        for i, b in enumerate(nb):
            lo, hi = b
            for d in range(2):
                n = hi[d] - lo[d] + 1
                assert 0 <= lo[d] <= hi[d] < dom[d]
                assert lo[d] % r[d] == 0 and (hi[d] + 1) % r[d] == 0          # refined coarse cells
                assert n <= largest[k][d] and (n >= smallest[k][d] or n == dom[d])
            for b2 in nb[i + 1:]:
                assert boxes.is_empty(boxes.intersect(b, b2))                   # disjoint
            # proper nesting: every coarsened cell lies in a level-k box
            cb = boxes.coarsen(b, r)
            covered = sum(boxes.ncells(boxes.intersect(cb, c)) for c in coarse)
            assert covered == boxes.ncells(cb)
