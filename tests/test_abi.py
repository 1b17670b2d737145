"""CPU tests of the C-ABI library: it loads, exports every symbol include/vlasov.h declares, and
its host-side metadata (layout, ghost maps, Alg.7 sub-patches, tile rule) matches the oracle
bit-exactly.  No compute call is made without a GPU (those must fail loudly with ECUDA)."""
import numpy as np
import pytest

import inputs
from inputs.hierarchies import random_hierarchy
from oracle import amr, boxes as obox

from paper_1204_3853_b200 import _lib, api


def test_library_exports_every_header_symbol():
    syms = _lib.header_symbols()
    assert len(syms) >= 20
    for s in syms:
        assert hasattr(_lib.lib, s), s
    assert _lib.lib.vlasov_version() >= 1


def _geom(w):
    return api.make_geom(w.ndim, w.ncells, w.lower, inputs.spacing(w))


def test_compute_calls_fail_loudly_without_device():
    if api.vlasov_device_ok():
        pytest.skip("device present")
    w = inputs.get("C1")
    lvl = api.Level(2, w.ncells, w.lower, inputs.spacing(w), (1, 1), inputs.level0_boxes(w))
    rc = _lib.lib.vlasov_rhs(lvl.h, None, None, None, 0)
    assert rc == _lib.EINVAL
    import ctypes as C
    buf = (C.c_double * 16)()
    rc = _lib.lib.vlasov_rhs(lvl.h, buf, buf, buf, 0)
    assert rc == _lib.ECUDA
    assert "device" in api.vlasov_last_error()


def test_invalid_boxes_rejected():
    w = inputs.get("C1")
    g = _geom(w)
    with pytest.raises(_lib.VlasovError) as e:
        api.vlasov_level_create(g, (1, 1), [((0, 0), (63, 63)), ((10, 10), (20, 20))])
    assert e.value.code == _lib.ENEST
    with pytest.raises(_lib.VlasovError) as e:
        api.vlasov_level_create(g, (1, 1), [((0, 0), (31, 63))])       # level 0 must tile the domain
    assert e.value.code == _lib.ENEST
    with pytest.raises(_lib.VlasovError) as e:
        api.vlasov_level_create(g, (1, 1), [((0, 0), (64, 63))])
    assert e.value.code == _lib.ENEST


def test_layout_merged_single_block():
    w = inputs.get("C4")
    lvl = api.Level(2, w.ncells, w.lower, inputs.spacing(w), (1, 1), inputs.level0_boxes(w))
    assert lvl.info.nblocks == 1 and lvl.info.npatches == 2048
    off0, st = lvl.layouts[0]
    pitch = st[0]
    assert st[1] == 1 and pitch >= 4096 + 4 and pitch % 2 == 0
    assert off0 == 2 * pitch + 2
    # patch (i, j) interior origin sits at row 64 i, column 64 j of the merged block
    p = 5 * 64 + 7
    lo, _ = lvl.boxes[p]
    assert lvl.layouts[p][0] == (lo[0] + 2) * pitch + lo[1] + 2
    assert lvl.info.ntiles >= 16 and lvl.info.ntiles % 16 == 0        # 16 v-tiles of 256 per row strip


def _api_hierarchy(rat, lb, w):
    levels = []
    for l, (r, bl) in enumerate(zip(rat, lb)):
        levels.append(api.Level(2, w.ncells, w.lower, inputs.spacing(w), r, bl,
                                coarser=levels[-1] if levels else None))
    return levels


@pytest.mark.parametrize("seed", range(15))
def test_ghost_maps_bitexact_vs_oracle(seed):
    w = inputs.scaled(inputs.get("C3"), (16, 32), (8, 8))
    rat, lb = random_hierarchy(seed)
    levels = _api_hierarchy(rat, lb, w)
    dom = obox.box((0, 0), (15, 31))
    metas = [obox.LevelMeta(dom, r, [obox.box(*b) for b in bl], (True, False)) for r, bl in zip(rat, lb)]
    for l, L in enumerate(levels):
        for p, (lo, hi) in enumerate(L.boxes):
            n = (hi[0] - lo[0] + 5) * (hi[1] - lo[1] + 5)
            k, sp, sc = api.vlasov_level_ghost_map(L.h, p, n)
            ok, osp, osc = obox.ghost_map(metas[l], p, metas[l - 1] if l else None)
            assert np.array_equal(k, ok) and np.array_equal(sp, osp) and np.array_equal(sc, osc)


@pytest.mark.parametrize("seed", range(15))
def test_subpatches_bitexact_vs_oracle(seed):
    w = inputs.scaled(inputs.get("C3"), (16, 32), (8, 8))
    rat, lb = random_hierarchy(seed)
    levels = _api_hierarchy(rat, lb, w)
    dom = obox.box((0, 0), (15, 31))
    metas = [obox.LevelMeta(dom, r, [obox.box(*b) for b in bl], (True, False)) for r, bl in zip(rat, lb)]
    hs = [L.h for L in levels]
    for l, L in enumerate(levels):
        for p, b in enumerate(L.boxes):
            got = api.vlasov_subpatches(hs, l, p)
            exp = obox.compute_sub_patches(obox.box(*b), l, metas)
            got2 = [(lo[:2], hi[:2]) for lo, hi in got]
            assert got2 == [(tuple(e[0]), tuple(e[1])) for e in exp]


def test_tile_rule_bitexact_vs_oracle():
    rng = np.random.default_rng(0)
    for trial in range(20):
        tags = rng.random((128, 256)) < 0.002
        d = obox.dilate_tags(tags, 1, (True, False))
        got = api.vlasov_tags_to_boxes(d.astype(np.uint8), (128, 256), (4, 4), 32)
        exp = obox.tiles_from_tags(d, (4, 4), 32)
        assert got == [(tuple(b[0]), tuple(b[1])) for b in exp]
