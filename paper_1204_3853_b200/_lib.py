"""ctypes loader for the in-tree libvlasov.so (built by ``__graft_entry__.build()``).

Argument marshalling only.  There is no fallback: if the shared library is missing the import
fails loudly, and every compute entry point reports VLASOV_ECUDA without an sm_100 device.
"""
from __future__ import annotations

import ctypes as C
import os
import re

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "libvlasov.so")
HEADER = os.path.join(os.path.dirname(HERE), "include", "vlasov.h")

OK, EINVAL, ENOMEM, ECUDA, ENEST, ESTALE, ESTENCIL, EUNSUPPORTED = 0, -1, -2, -3, -4, -5, -6, -7
CENTERED4, UPWIND = 0, 1
LINEAR5, WENO5 = 0, 1
GHOST_INTERIOR, GHOST_SIBLING, GHOST_COARSE, GHOST_PHYS = 0, 1, 2, 3


class VlasovError(RuntimeError):
    def __init__(self, code, msg):
        super().__init__(f"libvlasov error {code}: {msg}")
        self.code = code


class Box(C.Structure):
    _fields_ = [("lo", C.c_int32 * 4), ("hi", C.c_int32 * 4)]


class Geom(C.Structure):
    _fields_ = [("ndim", C.c_int32), ("domain", Box), ("lower", C.c_double * 4), ("dx0", C.c_double * 4)]


class LevelInfo(C.Structure):
    _fields_ = [("field_doubles", C.c_int64), ("e_doubles", C.c_int64), ("cfg_cells", C.c_int64),
                ("fluxreg_doubles", C.c_int64), ("tag_bytes", C.c_int64),
                ("nblocks", C.c_int32), ("npatches", C.c_int32), ("ntiles", C.c_int32), ("ndim", C.c_int32),
                ("ratio", C.c_int32 * 4), ("ncfg", C.c_int32 * 2), ("domain_cells", C.c_int32 * 4)]


if not os.path.exists(LIB_PATH):
    raise ImportError(f"{LIB_PATH} not built: run `python -c 'import __graft_entry__ as g; g.build()'`")

lib = C.CDLL(LIB_PATH)

P = C.c_void_p
I32 = C.c_int32
I64 = C.c_int64
D = C.c_double
PI32 = C.POINTER(C.c_int32)
PI64 = C.POINTER(C.c_int64)

_SIGS = {
    "vlasov_level_create": (I32, [C.POINTER(Geom), PI32, C.POINTER(Box), I32, P, P, C.POINTER(P)]),
    "vlasov_level_destroy": (I32, [P]),
    "vlasov_level_get_info": (I32, [P, C.POINTER(LevelInfo)]),
    "vlasov_level_layout": (I32, [P, I32, PI64, PI64]),
    "vlasov_level_ghost_map": (I32, [P, I32, PI32, PI32, PI64]),
    "vlasov_subpatches": (I32, [C.POINTER(P), I32, I32, I32, C.POINTER(Box), I32, PI32]),
    "vlasov_fill_ghosts": (I32, [P, P, P, P, P, P, I32]),
    "vlasov_rhs": (I32, [P, P, P, P, I32]),
    "vlasov_rk4_stage": (I32, [P, I32, D, P, P, P, P, P, P, P, I32, P]),
    "vlasov_rk4_stage_vp": (I32, [P, P, I32, D, P, P, P, P, P, P, P, P, I32, P]),
    "vlasov_reduce_moment": (I32, [C.POINTER(P), I32, C.POINTER(P), P]),
    "vlasov_reduce_moment_mask": (I32, [C.POINTER(P), I32, C.POINTER(P), P]),
    "vlasov_reduce_charge": (I32, [C.POINTER(P), I32, C.POINTER(P), D, D, I32, P]),
    "vlasov_inject_field_scaled": (I32, [P, P, PI32, D, P]),
    "vlasov_absmax": (I32, [P, I64, P, P]),
    "vlasov_next_dt": (I32, [C.POINTER(P), I32, C.POINTER(P), D, D, D, C.POINTER(D)]),
    "vlasov_level_set_moment_base": (I32, [P, D]),
    "vlasov_level_set_velocity_faces": (I32, [P, I32, I32]),
    "vlasov_reduce_current": (I32, [P, I32, P, D, I32, P]),
    "vlasov_vslab_pack": (I32, [P, P, P, P]),
    "vlasov_vslab_unpack": (I32, [P, P, P, P]),
    "vlasov_poisson_create": (I32, [I32, D, P, C.POINTER(P)]),
    "vlasov_poisson_solve": (I32, [P, P, P, P, I32]),
    "vlasov_poisson_destroy": (I32, [P]),
    "vlasov_inject_field_ghosted": (I32, [P, P, PI32, P]),
    "vlasov_level_face_doubles": (I32, [P, PI64]),
    "vlasov_rk4_stage_fstar": (I32, [P, I32, D, P, P, P, P, I32, P]),
    "vlasov_fstar_coarsen": (I32, [P, P, P, P]),
    "vlasov_fstar_update": (I32, [P, D, P, P, P]),
    "vlasov_poisson2d_create": (I32, [I32, I32, D, D, P, C.POINTER(P)]),
    "vlasov_poisson2d_solve": (I32, [P, P, P]),
    "vlasov_poisson2d_destroy": (I32, [P]),
    "vlasov_inject_field": (I32, [P, P, PI32, P]),
    "vlasov_flux_register_accumulate": (I32, [P, P, P, P, P, D, P, I32]),
    "vlasov_average_down": (I32, [P, P, P, P, D]),
    "vlasov_tag_cells": (I32, [P, P, D, I32, P]),
    "vlasov_tags_to_boxes": (I32, [P, PI32, I32, PI32, I32, C.POINTER(Box), I32, PI32]),
    "vlasov_cluster_tags": (I32, [P, PI32, PI32, PI32, PI32, D, C.POINTER(Box), I32, PI32]),
    "vlasov_regrid_boxes": (I32, [P, P, PI32, PI32, PI32, D, I32, C.POINTER(Box), I32, PI32]),
    "vlasov_level_fill_from": (I32, [P, P, P, P, P, P, I32]),
    "vlasov_last_error": (C.c_char_p, []),
    "vlasov_device_ok": (I32, []),
    "vlasov_version": (I32, []),
}

for _name, (_res, _args) in _SIGS.items():
    _fn = getattr(lib, _name)
    _fn.restype = _res
    _fn.argtypes = _args


def header_symbols():
    """Function names declared in include/vlasov.h."""
    src = open(HEADER).read()
    return sorted(set(re.findall(r"\b(vlasov_[a-z0-9_]+)\s*\(", src)))


def check(rc):
    if rc != OK:
        raise VlasovError(rc, lib.vlasov_last_error().decode())
    return rc
