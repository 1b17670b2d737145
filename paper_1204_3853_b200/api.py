"""Thin Python binding of the libvlasov C ABI (include/vlasov.h): same names, argument marshalling
only.  Field arguments are torch CUDA float64 tensors (or None); every compute step runs in the
library's CUDA kernels on the level's stream.  PyTorch provides device memory and streams only.
"""
from __future__ import annotations

import ctypes as C
from typing import Optional, Sequence

import numpy as np
import torch

from . import _lib
from ._lib import Box, Geom, LevelInfo, check, lib

__all__ = [
    "Level", "Poisson", "make_geom", "vlasov_level_create", "vlasov_level_destroy",
    "vlasov_level_get_info", "vlasov_level_layout", "vlasov_level_ghost_map", "vlasov_subpatches",
    "vlasov_fill_ghosts", "vlasov_rhs", "vlasov_rk4_stage", "vlasov_rk4_stage_vp", "vlasov_reduce_moment", "vlasov_reduce_moment_mask", "vlasov_reduce_charge", "vlasov_inject_field_scaled",
    "vlasov_poisson_create", "vlasov_poisson_solve", "vlasov_poisson_destroy", "vlasov_inject_field",
    "vlasov_flux_register_accumulate", "vlasov_average_down", "vlasov_tag_cells", "vlasov_tags_to_boxes", "vlasov_cluster_tags", "vlasov_regrid_boxes",
    "vlasov_level_fill_from", "vlasov_absmax", "vlasov_next_dt", "vlasov_poisson2d_create",
    "vlasov_poisson2d_solve", "Poisson2D", "vlasov_inject_field_ghosted", "vlasov_level_face_doubles",
    "vlasov_rk4_stage_fstar", "vlasov_fstar_coarsen", "vlasov_fstar_update", "vlasov_device_ok", "vlasov_last_error",
    "vlasov_level_set_moment_base", "vlasov_level_set_velocity_faces", "vlasov_vslab_pack", "vlasov_vslab_unpack", "vlasov_reduce_current",
]


def _ptr(t: Optional[torch.Tensor]):
    if t is None:
        return None
    if not t.is_cuda:
        raise ValueError("libvlasov fields must be CUDA tensors")
    if t.dtype not in (torch.float64, torch.uint8):
        raise ValueError("libvlasov fields are float64 (tags: uint8)")
    if not t.is_contiguous():
        raise ValueError("libvlasov fields must be contiguous")
    return C.c_void_p(t.data_ptr())


def _stream_ptr(stream):
    if stream is None:
        return C.c_void_p(torch.cuda.current_stream().cuda_stream) if torch.cuda.is_available() else None
    return C.c_void_p(stream.cuda_stream if hasattr(stream, "cuda_stream") else int(stream))


def make_geom(ndim, ncells, lower, dx0) -> Geom:
    g = Geom()
    g.ndim = ndim
    for d in range(4):
        g.domain.lo[d] = 0
        g.domain.hi[d] = (ncells[d] - 1) if d < ndim else 0
        g.lower[d] = lower[d] if d < ndim else 0.0
        g.dx0[d] = dx0[d] if d < ndim else 0.0
    return g


def _boxes(boxes) -> C.Array:
    arr = (Box * len(boxes))()
    for i, (lo, hi) in enumerate(boxes):
        for d in range(4):
            arr[i].lo[d] = lo[d] if d < len(lo) else 0
            arr[i].hi[d] = hi[d] if d < len(hi) else 0
    return arr


# ----------------------------------------------------------------------------- raw names
def vlasov_level_create(geom, ratio, boxes, coarser=None, stream=None):
    out = C.c_void_p()
    r = (C.c_int32 * 4)(*(list(ratio) + [1] * (4 - len(ratio))))
    bx = _boxes(boxes)
    check(lib.vlasov_level_create(C.byref(geom), r, bx, len(boxes), coarser, _stream_ptr(stream), C.byref(out)))
    return out


def vlasov_level_destroy(h):
    return check(lib.vlasov_level_destroy(h))


def vlasov_level_get_info(h) -> LevelInfo:
    info = LevelInfo()
    check(lib.vlasov_level_get_info(h, C.byref(info)))
    return info


def vlasov_level_layout(h, patch):
    off = C.c_int64()
    st = (C.c_int64 * 4)()
    check(lib.vlasov_level_layout(h, patch, C.byref(off), st))
    return off.value, tuple(st)


def vlasov_level_ghost_map(h, patch, ncells_grown):
    kind = np.zeros(ncells_grown, np.int32)
    sp = np.zeros(ncells_grown, np.int32)
    sc = np.zeros(ncells_grown, np.int64)
    check(lib.vlasov_level_ghost_map(h, patch, kind.ctypes.data_as(_lib.PI32), sp.ctypes.data_as(_lib.PI32),
                                     sc.ctypes.data_as(_lib.PI64)))
    return kind, sp, sc


def vlasov_subpatches(levels, level_index, patch, cap=4096):
    arr = (C.c_void_p * len(levels))(*[l.value if isinstance(l, C.c_void_p) else l for l in levels])
    out = (Box * cap)()
    n = C.c_int32()
    check(lib.vlasov_subpatches(arr, len(levels), level_index, patch, out, cap, C.byref(n)))
    return [(tuple(out[i].lo), tuple(out[i].hi)) for i in range(min(n.value, cap))]


def vlasov_fill_ghosts(h, f, coarser=None, f_coarse=None, E_bc=None, f0v=None, interp=_lib.LINEAR5):
    return check(lib.vlasov_fill_ghosts(h, _ptr(f), coarser, _ptr(f_coarse), _ptr(E_bc), _ptr(f0v), interp))


def vlasov_rhs(h, f, E, k, recon=_lib.CENTERED4):
    return check(lib.vlasov_rhs(h, _ptr(f), _ptr(E), _ptr(k), recon))


def vlasov_rk4_stage(h, stage, dt, f_n, f_s, u, f_next, E, E_bc=None, f0v=None, recon=_lib.CENTERED4,
                     rho_next=None):
    return check(lib.vlasov_rk4_stage(h, stage, float(dt), _ptr(f_n), _ptr(f_s), _ptr(u), _ptr(f_next), _ptr(E),
                                      _ptr(E_bc), _ptr(f0v), recon, _ptr(rho_next)))


def vlasov_rk4_stage_vp(h, plan, stage, dt, f_n, f_s, u, f_next, rho_s, E_s, E_bc, f0v, recon=_lib.CENTERED4,
                        rho_next=None):
    return check(lib.vlasov_rk4_stage_vp(h, plan, stage, float(dt), _ptr(f_n), _ptr(f_s), _ptr(u), _ptr(f_next),
                                         _ptr(rho_s), _ptr(E_s), _ptr(E_bc), _ptr(f0v), recon, _ptr(rho_next)))


def vlasov_reduce_moment(levels, f_list, rho_finest):
    arr = (C.c_void_p * len(levels))(*[l.value if isinstance(l, C.c_void_p) else l for l in levels])
    fp = (C.c_void_p * len(levels))(*[(t.data_ptr() if t is not None else None) for t in f_list])
    return check(lib.vlasov_reduce_moment(arr, len(levels), fp, _ptr(rho_finest)))


def vlasov_reduce_current(levels, f_list, q, accumulate, j):
    """levels / f_list: one level handle and its field, or the hierarchy's lists (coarse first)."""
    if not isinstance(levels, (list, tuple)):
        levels, f_list = [levels], [f_list]
    arr = (C.c_void_p * len(levels))(*[l.value if isinstance(l, C.c_void_p) else l for l in levels])
    fp = (C.c_void_p * len(levels))(*[t.data_ptr() for t in f_list])
    return check(lib.vlasov_reduce_current(arr, len(levels), fp, float(q), int(bool(accumulate)), _ptr(j)))


def vlasov_level_set_moment_base(h, base):
    return check(lib.vlasov_level_set_moment_base(h, float(base)))


def vlasov_level_set_velocity_faces(h, phys_lo, phys_hi):
    return check(lib.vlasov_level_set_velocity_faces(h, int(bool(phys_lo)), int(bool(phys_hi))))


def vlasov_vslab_pack(h, f, lo=None, hi=None):
    return check(lib.vlasov_vslab_pack(h, _ptr(f), _ptr(lo), _ptr(hi)))


def vlasov_vslab_unpack(h, f, lo=None, hi=None):
    return check(lib.vlasov_vslab_unpack(h, _ptr(f), _ptr(lo), _ptr(hi)))


def vlasov_absmax(x, out, stream=None):
    return check(lib.vlasov_absmax(_ptr(x), x.numel(), _ptr(out), _stream_ptr(stream)))


def vlasov_next_dt(levels, E_list, dt_prev, cfl=0.5, growth=1.1):
    """Adaptive time step of a 1D+1V hierarchy (levels coarse first, E_list their ghosted E arrays)."""
    arr = (C.c_void_p * len(levels))(*[l.value if isinstance(l, C.c_void_p) else l for l in levels])
    ep = (C.c_void_p * len(levels))(*[t.data_ptr() for t in E_list])
    out = C.c_double(0.0)
    check(lib.vlasov_next_dt(arr, len(levels), ep, float(dt_prev), float(cfl), float(growth), C.byref(out)))
    return out.value


def vlasov_reduce_charge(levels, f_list, q, base, accumulate, rho_finest):
    arr = (C.c_void_p * len(levels))(*[l.value if isinstance(l, C.c_void_p) else l for l in levels])
    fp = (C.c_void_p * len(levels))(*[(t.data_ptr() if t is not None else None) for t in f_list])
    return check(lib.vlasov_reduce_charge(arr, len(levels), fp, float(q), float(base), int(accumulate),
                                          _ptr(rho_finest)))


def vlasov_inject_field_scaled(h, E_finest, n_finest, scale, E_lvl):
    n = (C.c_int32 * 2)(*(list(n_finest) + [1] * (2 - len(n_finest))))
    return check(lib.vlasov_inject_field_scaled(h, _ptr(E_finest), n, float(scale), _ptr(E_lvl)))


def vlasov_reduce_moment_mask(levels, f_list, rho_finest):
    arr = (C.c_void_p * len(levels))(*[l.value if isinstance(l, C.c_void_p) else l for l in levels])
    fp = (C.c_void_p * len(levels))(*[(t.data_ptr() if t is not None else None) for t in f_list])
    return check(lib.vlasov_reduce_moment_mask(arr, len(levels), fp, _ptr(rho_finest)))


def vlasov_poisson_create(n, dx, stream=None):
    out = C.c_void_p()
    check(lib.vlasov_poisson_create(n, float(dx), _stream_ptr(stream), C.byref(out)))
    return out


def vlasov_poisson_solve(p, rho, phi=None, E=None, ghost=0):
    return check(lib.vlasov_poisson_solve(p, _ptr(rho), _ptr(phi), _ptr(E), int(ghost)))


def vlasov_poisson_destroy(p):
    return check(lib.vlasov_poisson_destroy(p))


def vlasov_inject_field(h, E_finest, n_finest, E_lvl):
    n = (C.c_int32 * 2)(*(list(n_finest) + [1] * (2 - len(n_finest))))
    return check(lib.vlasov_inject_field(h, _ptr(E_finest), n, _ptr(E_lvl)))


def vlasov_flux_register_accumulate(fine, f_fine, E_fine, f_coarse, E_coarse, b_s, regs, recon=_lib.CENTERED4):
    return check(lib.vlasov_flux_register_accumulate(fine, _ptr(f_fine), _ptr(E_fine), _ptr(f_coarse),
                                                     _ptr(E_coarse), float(b_s), _ptr(regs), recon))


def vlasov_average_down(fine, f_fine, f_coarse, regs, dt):
    return check(lib.vlasov_average_down(fine, _ptr(f_fine), _ptr(f_coarse), _ptr(regs), float(dt)))


def vlasov_tag_cells(h, f, tol, buffer, tags):
    return check(lib.vlasov_tag_cells(h, _ptr(f), float(tol), int(buffer), _ptr(tags)))


def vlasov_tags_to_boxes(tags_host: np.ndarray, domain_cells, ratio, tile, cap=65536):
    t = np.ascontiguousarray(tags_host, dtype=np.uint8)
    dc = (C.c_int32 * 4)(*(list(domain_cells) + [0] * (4 - len(domain_cells))))
    r = (C.c_int32 * 4)(*(list(ratio) + [1] * (4 - len(ratio))))
    out = (Box * cap)()
    n = C.c_int32()
    check(lib.vlasov_tags_to_boxes(t.ctypes.data_as(C.c_void_p), dc, len(domain_cells), r, tile, out, cap,
                                   C.byref(n)))
    return [(tuple(out[i].lo[:2]), tuple(out[i].hi[:2])) for i in range(min(n.value, cap))]


def vlasov_cluster_tags(tags_host: np.ndarray, smallest, largest, efficiency=0.7, lo=(0, 0), cap=65536):
    t = np.ascontiguousarray(tags_host, dtype=np.uint8)
    sh = (C.c_int32 * 2)(*t.shape)
    l = (C.c_int32 * 2)(*lo)
    sm = (C.c_int32 * 2)(*smallest)
    lg = (C.c_int32 * 2)(*largest)
    out = (Box * cap)()
    n = C.c_int32()
    check(lib.vlasov_cluster_tags(t.ctypes.data_as(C.c_void_p), sh, l, sm, lg, float(efficiency), out, cap,
                                  C.byref(n)))
    return [(tuple(out[i].lo[:2]), tuple(out[i].hi[:2])) for i in range(min(n.value, cap))]


def vlasov_regrid_boxes(h, tags_host: np.ndarray, ratio, smallest, largest, efficiency=0.7, nest=1, cap=65536):
    t = np.ascontiguousarray(tags_host, dtype=np.uint8)
    r = (C.c_int32 * 2)(*ratio)
    sm = (C.c_int32 * 2)(*smallest)
    lg = (C.c_int32 * 2)(*largest)
    out = (Box * cap)()
    n = C.c_int32()
    check(lib.vlasov_regrid_boxes(h, t.ctypes.data_as(C.c_void_p), r, sm, lg, float(efficiency), int(nest), out, cap,
                                  C.byref(n)))
    return [(tuple(out[i].lo[:2]), tuple(out[i].hi[:2])) for i in range(min(n.value, cap))]


def vlasov_level_fill_from(h, f, old=None, f_old=None, coarser=None, f_coarse=None, interp=_lib.LINEAR5):
    return check(lib.vlasov_level_fill_from(h, _ptr(f), old, _ptr(f_old), coarser, _ptr(f_coarse), interp))


def vlasov_device_ok() -> bool:
    return bool(lib.vlasov_device_ok())


def vlasov_last_error() -> str:
    return lib.vlasov_last_error().decode()


# ----------------------------------------------------------------------------- objects
class Level:
    """Owns one vlasov_level handle; helpers to allocate fields and view patches."""

    def __init__(self, ndim, ncells0, lower, dx0, ratio, boxes, coarser: Optional["Level"] = None, stream=None):
        self.geom = make_geom(ndim, ncells0, lower, dx0)
        self.ndim = ndim
        self.ratio = tuple(ratio)
        self.boxes = [(tuple(lo), tuple(hi)) for lo, hi in boxes]
        self.coarser = coarser
        self.h = vlasov_level_create(self.geom, ratio, self.boxes, coarser.h if coarser else None, stream)
        self.info = vlasov_level_get_info(self.h)
        self._layouts = None

    @property
    def layouts(self):
        """Per-patch (offset, strides), queried on first use (a regrid's new level needs none)."""
        if self._layouts is None:
            self._layouts = [vlasov_level_layout(self.h, p) for p in range(len(self.boxes))]
        return self._layouts

    def __del__(self):
        try:
            if getattr(self, "h", None):
                lib.vlasov_level_destroy(self.h)
                self.h = None
        except Exception:
            pass

    def field(self, fill=float("nan")):
        return torch.full((self.info.field_doubles,), fill, dtype=torch.float64, device="cuda")

    def efield(self):
        return torch.zeros(self.info.e_doubles, dtype=torch.float64, device="cuda")

    def patch_view(self, f: torch.Tensor, p: int, ghost: int = 0):
        off, st = self.layouts[p]
        lo, hi = self.boxes[p]
        size = [hi[d] - lo[d] + 1 + 2 * ghost for d in range(self.ndim)]
        start = off - sum(ghost * st[d] for d in range(self.ndim))
        return torch.as_strided(f, size, st[:self.ndim], start)

    def set_patches(self, f: torch.Tensor, arrays):
        for p, a in enumerate(arrays):
            self.patch_view(f, p).copy_(torch.as_tensor(a, dtype=torch.float64))

    def get_patches(self, f: torch.Tensor, ghost: int = 0):
        return [self.patch_view(f, p, ghost).cpu().numpy() for p in range(len(self.boxes))]

    def _covers_domain_as_one_block(self):
        return self.info.nblocks == 1 and all(
            min(b[0][d] for b in self.boxes) == 0 and max(b[1][d] for b in self.boxes) == self.info.domain_cells[d] - 1
            for d in range(self.ndim))

    def set_domain(self, f: torch.Tensor, full: np.ndarray):
        """Scatter a whole-domain array (level index space) into the patches."""
        if self._covers_domain_as_one_block():
            g = [slice(2, -2)] * self.ndim
            self.block_view(f, 2)[tuple(g)].copy_(torch.as_tensor(np.ascontiguousarray(full)))
            return
        for p, (lo, hi) in enumerate(self.boxes):
            sl = tuple(slice(lo[d], hi[d] + 1) for d in range(self.ndim))
            self.patch_view(f, p).copy_(torch.as_tensor(np.ascontiguousarray(full[sl])))

    def block_view(self, f: torch.Tensor, ghost: int = 2):
        """Whole ghosted block of a single-block level."""
        assert self.info.nblocks == 1
        off, st = self.layouts[0]
        lo, _ = self.boxes[0]
        lo_all = [min(b[0][d] for b in self.boxes) for d in range(self.ndim)]
        hi_all = [max(b[1][d] for b in self.boxes) for d in range(self.ndim)]
        start = off - sum((lo[d] - lo_all[d] + ghost) * st[d] for d in range(self.ndim))
        size = [hi_all[d] - lo_all[d] + 1 + 2 * ghost for d in range(self.ndim)]
        return torch.as_strided(f, size, st[:self.ndim], start)

    def get_domain(self, f: torch.Tensor) -> np.ndarray:
        if self._covers_domain_as_one_block():
            g = [slice(2, -2)] * self.ndim
            return self.block_view(f, 2)[tuple(g)].cpu().numpy()
        out = np.full(tuple(self.info.domain_cells[d] for d in range(self.ndim)), np.nan)
        for p, (lo, hi) in enumerate(self.boxes):
            sl = tuple(slice(lo[d], hi[d] + 1) for d in range(self.ndim))
            out[sl] = self.patch_view(f, p).cpu().numpy()
        return out


class Poisson:
    def __init__(self, n, dx, stream=None):
        self.n = n
        self.h = vlasov_poisson_create(n, dx, stream)

    def solve(self, rho, phi=None, E=None, ghost=0):
        vlasov_poisson_solve(self.h, rho, phi, E, ghost)

    def __del__(self):
        try:
            if getattr(self, "h", None):
                lib.vlasov_poisson_destroy(self.h)
                self.h = None
        except Exception:
            pass


def vlasov_poisson2d_create(nx, ny, dx, dy, stream=None):
    h = C.c_void_p()
    check(lib.vlasov_poisson2d_create(int(nx), int(ny), float(dx), float(dy), _stream_ptr(stream), C.byref(h)))
    return h


def vlasov_poisson2d_solve(h, rho, E):
    return check(lib.vlasov_poisson2d_solve(h, _ptr(rho), _ptr(E)))


class Poisson2D:
    """2D periodic field plan (N3, reading #32): rho (nx ny) -> ghosted E [2][(nx+4)(ny+4)]."""

    def __init__(self, nx, ny, dx, dy, stream=None):
        self.nx, self.ny = nx, ny
        self.h = vlasov_poisson2d_create(nx, ny, dx, dy, stream)

    def solve(self, rho, E):
        vlasov_poisson2d_solve(self.h, rho, E)

    def __del__(self):
        try:
            if getattr(self, "h", None):
                lib.vlasov_poisson2d_destroy(self.h)
                self.h = None
        except Exception:
            pass


def vlasov_inject_field_ghosted(h, E_finest, n_finest, E_lvl):
    n = (C.c_int32 * 2)(*n_finest)
    return check(lib.vlasov_inject_field_ghosted(h, _ptr(E_finest), n, _ptr(E_lvl)))


def vlasov_level_face_doubles(h):
    n = C.c_int64()
    check(lib.vlasov_level_face_doubles(h, C.byref(n)))
    return n.value


def vlasov_rk4_stage_fstar(h, stage, dt, f_n, f_s, f_next, E, recon, Fstar):
    return check(lib.vlasov_rk4_stage_fstar(h, int(stage), float(dt), _ptr(f_n), _ptr(f_s), _ptr(f_next), _ptr(E),
                                            int(recon), _ptr(Fstar)))


def vlasov_fstar_coarsen(fine, F_fine, coarse, F_coarse):
    return check(lib.vlasov_fstar_coarsen(fine, _ptr(F_fine), coarse, _ptr(F_coarse)))


def vlasov_fstar_update(h, dt, f_n, Fstar, f_new):
    return check(lib.vlasov_fstar_update(h, float(dt), _ptr(f_n), _ptr(Fstar), _ptr(f_new)))
