"""Error behaviour of the C ABI (include/vlasov.h "Status"): argument validation happens before
any device work, so every check here runs on the CPU-only host; compute entry points without an
sm_100 device fail loudly with VLASOV_ECUDA (never a silent CPU fallback)."""
import ctypes as C

import numpy as np
import pytest

import inputs
from paper_1204_3853_b200 import _lib, api

lib = _lib.lib


def _geom(ndim=2, ncells=(16, 32)):
    lower = (0.0,) * ndim
    dx = (0.1,) * ndim
    return api.make_geom(ndim, ncells, lower, dx)


def _create(geom, ratio, boxes, coarser=None):
    out = C.c_void_p()
    r = (C.c_int32 * 4)(*(list(ratio) + [1] * (4 - len(ratio))))
    bx = api._boxes(boxes) if boxes else (_lib.Box * 1)()
    rc = lib.vlasov_level_create(C.byref(geom), r, bx, len(boxes), coarser, None, C.byref(out))
    return rc, out


def test_create_argument_errors():
    g = _geom()
    assert _create(g, (1, 1), [])[0] == _lib.EINVAL                                 # nboxes < 1
    assert _create(g, (0, 1), [((0, 0), (15, 31))])[0] == _lib.EINVAL               # ratio < 1
    assert _create(g, (1, 1), [((3, 0), (2, 31))])[0] == _lib.EINVAL                # empty box
    assert _create(g, (1, 1), [((0, 0), (16, 31))])[0] == _lib.ENEST                # outside the domain
    g3 = _geom()
    g3.ndim = 3
    assert _create(g3, (1, 1, 1), [((0, 0, 0), (1, 1, 1))])[0] == _lib.EINVAL        # ndim must be 2 or 4
    rc = lib.vlasov_level_create(None, None, None, 0, None, None, None)
    assert rc == _lib.EINVAL
    assert "null" in api.vlasov_last_error()


def test_nesting_and_alignment_errors():
    g = _geom()
    rc, L0 = _create(g, (1, 1), [((0, 0), (15, 31))])
    assert rc == _lib.OK
    # fine box whose coarse parents leave the coarser level: not possible on a tiling level 0,
    # so use a coarser level made of one patch and a fine box outside it
    rc, Lp = _create(g, (2, 2), [((0, 0), (7, 15))], L0)
    assert rc == _lib.OK
    rc, _ = _create(g, (4, 4), [((40, 40), (47, 47))], Lp)
    assert rc == _lib.ENEST
    # fine boxes not aligned to coarse cells (flux registers need whole coarse faces)
    rc, _ = _create(g, (2, 2), [((1, 2), (6, 9))], L0)
    assert rc == _lib.EINVAL
    # coarser level with another ndim / ratio not a multiple
    rc, _ = _create(g, (3, 2), [((0, 0), (5, 5))], Lp)
    assert rc == _lib.EINVAL
    for h in (Lp, L0):
        lib.vlasov_level_destroy(h)


def test_compute_entry_points_validate_then_need_a_device():
    g = _geom()
    rc, L = _create(g, (1, 1), [((0, 0), (15, 31))])
    assert rc == _lib.OK
    buf = (C.c_double * 64)()
    nxt = (C.c_double * 64)()
    # validation errors first
    assert lib.vlasov_rk4_stage(L, 0, 0.1, buf, buf, buf, buf, buf, None, None, 0, None) == _lib.EINVAL
    assert lib.vlasov_rk4_stage(L, 2, 0.1, None, buf, buf, buf, buf, None, None, 0, None) == _lib.EINVAL
    assert lib.vlasov_rk4_stage(L, 1, 0.1, buf, buf, buf, buf, buf, None, None, 7, None) == _lib.EINVAL
    assert lib.vlasov_rk4_stage(L, 1, 0.1, buf, buf, buf, buf, buf, buf, None, 0, None) == _lib.EINVAL
    # f_next aliasing f_s: neighbouring CTAs read halo rows of f_s (a cross-CTA race)
    assert lib.vlasov_rk4_stage(L, 2, 0.1, buf, buf, buf, buf, buf, None, None, 0, None) == _lib.EINVAL
    assert lib.vlasov_tag_cells(L, buf, 0.1, -1, buf) == _lib.EINVAL
    assert lib.vlasov_average_down(L, buf, buf, None, 0.1) == _lib.EINVAL           # no coarser level
    P = C.c_void_p()
    assert lib.vlasov_poisson_create(4, 0.1, None, C.byref(P)) == _lib.EINVAL        # n >= 5
    assert lib.vlasov_poisson_create(16, -1.0, None, C.byref(P)) == _lib.EINVAL
    Ls = (C.c_void_p * 1)(L)
    fs = (C.c_void_p * 1)(C.cast(buf, C.c_void_p))
    assert lib.vlasov_reduce_current(Ls, 0, fs, -1.0, 0, buf) == _lib.EINVAL       # nlev >= 1
    assert lib.vlasov_reduce_current(Ls, 1, fs, -1.0, 0, None) == _lib.EINVAL     # j required
    assert lib.vlasov_reduce_current(Ls, 1, (C.c_void_p * 1)(None), -1.0, 0, buf) == _lib.EINVAL
    dto = C.c_double()
    assert lib.vlasov_next_dt(Ls, 0, fs, 0.01, 0.5, 1.1, C.byref(dto)) == _lib.EINVAL      # nlev >= 1
    assert lib.vlasov_next_dt(Ls, 1, fs, 0.01, 0.0, 1.1, C.byref(dto)) == _lib.EINVAL      # cfl > 0
    assert lib.vlasov_next_dt(Ls, 1, fs, -1.0, 0.5, 1.1, C.byref(dto)) == _lib.EINVAL      # dt_prev > 0
    assert lib.vlasov_next_dt(Ls, 1, fs, 0.01, 0.5, 1.1, None) == _lib.EINVAL              # output required
    if not api.vlasov_device_ok():
        assert lib.vlasov_reduce_current(Ls, 1, fs, -1.0, 0, buf) == _lib.ECUDA
        assert lib.vlasov_rk4_stage(L, 1, 0.1, buf, buf, buf, nxt, buf, None, None, 0, None) == _lib.ECUDA
        assert lib.vlasov_fill_ghosts(L, buf, None, None, buf, buf, 0) == _lib.ECUDA
        assert lib.vlasov_inject_field(L, buf, (C.c_int32 * 2)(16, 1), buf) == _lib.ECUDA
        assert lib.vlasov_poisson_create(16, 0.1, None, C.byref(P)) in (_lib.ECUDA, _lib.OK)
    lib.vlasov_level_destroy(L)


def test_2d2v_level_requirements():
    g = _geom(4, (8, 8, 12, 16))
    assert _create(g, (1, 1, 1, 1), [((0, 0, 0, 0), (7, 7, 11, 15))])[0] == _lib.OK
    g2 = _geom(4, (8, 8, 10, 16))                                                    # nvx % 4 != 0
    assert _create(g2, (1, 1, 1, 1), [((0, 0, 0, 0), (7, 7, 9, 15))])[0] == _lib.EINVAL
    g3 = _geom(4, (8, 8, 12, 16))                                                    # not tiling the domain
    assert _create(g3, (1, 1, 1, 1), [((0, 0, 0, 0), (3, 7, 11, 15))])[0] in (_lib.EUNSUPPORTED, _lib.ENEST)


def test_tags_to_boxes_errors_and_empty():
    t = np.zeros((8, 16), np.uint8)
    assert api.vlasov_tags_to_boxes(t, (8, 16), (4, 4), 16) == []                   # no tags -> no boxes
    with pytest.raises(_lib.VlasovError):
        api.vlasov_tags_to_boxes(t, (8, 16), (4, 4), 6)                               # tile not a ratio multiple
