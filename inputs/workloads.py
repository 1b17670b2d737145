"""Workload definitions C1-C5 (BASELINE.json ``configs``) and their inputs.

Everything here is problem SETUP, not the discretisation of PAPER.md section 2:

* geometry (domain, cell counts, level-0 patch tiling),
* exact cell averages of the initial distribution functions, computed in
  closed form with erf (BASELINE.json configs; bump profile P:1455-1461 shape
  with BASELINE.json's parameters, SURVEY.md section 8(c) reading #23),
* exact cell averages of the *unperturbed* velocity profile that the
  characteristic boundary condition injects on incoming characteristics
  ("incoming characteristics carry values from an unperturbed
  Maxwellian distribution"),
* the prescribed C5 field E(x, y) = 0.1 (cos x, sin y) as exact 2D cell
  averages (BASELINE.json C5),
* a fixed time step chosen from a CFL number of 0.5 (BASELINE.json C1) using the
  continuum linear-field amplitude bound alpha*mass/k, and
* seeded random arrays for parity tests.

Index convention: configuration dims first, then velocity dims;
the last (velocity) dim is contiguous.
"""
from __future__ import annotations

import math
from dataclasses import dataclass, field
from typing import Optional, Sequence, Tuple

import numpy as np
from scipy import special

__all__ = [
    "Workload", "WORKLOADS", "get", "spacing", "level0_boxes", "cell_edges",
    "initial_cell_averages", "background_profile", "prescribed_field",
    "fixed_dt", "random_field", "random_positive_field", "GHOST", "scaled",
]

GHOST = 2  # ghost width used by both sides (SURVEY.md 8(c) reading #7)

SQRT2 = math.sqrt(2.0)


@dataclass(frozen=True)
class Workload:
    name: str
    ncfg: int                      # 1 (1D+1V) or 2 (2D+2V)
    ncells: Tuple[int, ...]        # level-0 cells per dim
    lower: Tuple[float, ...]
    upper: Tuple[float, ...]
    patch: Tuple[int, ...]         # level-0 patch size per dim
    ic: str                        # 'landau' | 'twostream' | 'bump' | 'landau2d'
    alpha: float                   # perturbation amplitude
    k: Tuple[float, ...]           # perturbation wavenumbers per config dim
    field: str                     # 'poisson' | 'prescribed'
    steps: int
    amr: Optional[dict] = None     # C3 only
    description: str = ""

    @property
    def ndim(self) -> int:
        return len(self.ncells)

    @property
    def cells(self) -> int:
        return int(np.prod(self.ncells))


FOUR_PI = 4.0 * math.pi

WORKLOADS = {
    "C1": Workload(
        "C1", 1, (64, 64), (0.0, -6.0), (FOUR_PI, 6.0), (64, 64), "landau", 0.01,
        (0.5,), "poisson", 50,
        description="1D+1V Landau, single uniform patch 64x64, x in [0,4pi), v in [-6,6]"),
    "C2": Workload(
        "C2", 1, (256, 512), (0.0, -8.0), (FOUR_PI, 8.0), (256, 512), "landau", 0.01,
        (0.5,), "poisson", 1000,
        description="1D+1V linear Landau damping, uniform 256x512, v in [-8,8]"),
    "C3": Workload(
        "C3", 1, (128, 256), (0.0, -8.0), (FOUR_PI, 8.0), (32, 32), "twostream", 0.05,
        (0.5,), "poisson", 100,
        amr={"ratio": (4, 4), "tile": 32, "tol": 0.005, "buffer": 1, "regrid": 10},
        description="1D+1V two-stream, 2-level AMR, base 128x256, ratio 4, 32x32 fine tiles"),
    "C4": Workload(
        "C4", 1, (2048, 4096), (0.0, -10.0), (20.0 * math.pi / 3.0, 10.0), (64, 64), "bump",
        0.04, (0.3,), "poisson", 100,
        description="1D+1V bump-on-tail, uniform 2048x4096 (64x64 patches)"),
    "C5": Workload(
        "C5", 2, (64, 64, 64, 64), (0.0, 0.0, -6.0, -6.0),
        (2 * math.pi, 2 * math.pi, 6.0, 6.0), (16, 16, 16, 16), "landau2d", 0.01,
        (1.0, 1.0), "prescribed", 50,
        description="2D+2V stress case, 64^4 in 16^4 patches, prescribed E=0.1(cos x, sin y)"),
    # NEXT row N3 (not a BASELINE.json config): the C5 geometry and initial data with the
    # self-consistent field of the 2D periodic Poisson problem (reading #32) instead of the
    # prescribed one; the 2D+2V AMR tests use scaled-down versions of it
    "C5P": Workload(
        "C5P", 2, (64, 64, 64, 64), (0.0, 0.0, -6.0, -6.0),
        (2 * math.pi, 2 * math.pi, 6.0, 6.0), (16, 16, 16, 16), "landau2d", 0.01,
        (1.0, 1.0), "poisson", 50,
        description="N3: 2D+2V Vlasov-Poisson, C5 geometry, self-consistent 2D periodic field"),
}


def get(name: str) -> Workload:
    return WORKLOADS[name]


def scaled(w: Workload, ncells: Sequence[int], patch: Optional[Sequence[int]] = None,
           name: Optional[str] = None) -> Workload:
    """Same physics on a different grid (used for small parity cases)."""
    from dataclasses import replace
    return replace(w, ncells=tuple(int(n) for n in ncells),
                   patch=tuple(int(p) for p in (patch if patch is not None else ncells)),
                   name=name or f"{w.name}@{'x'.join(map(str, ncells))}")


def spacing(w: Workload, ratio: Sequence[int] = None) -> Tuple[float, ...]:
    ratio = ratio or (1,) * w.ndim
    return tuple((w.upper[d] - w.lower[d]) / (w.ncells[d] * ratio[d]) for d in range(w.ndim))


def cell_edges(w: Workload, d: int, ratio: int = 1, lo: int = None, hi: int = None) -> np.ndarray:
    """Edges x_{i-1/2} for cells lo..hi (inclusive) of dim d at refinement ``ratio``."""
    n = w.ncells[d] * ratio
    lo = 0 if lo is None else lo
    hi = n - 1 if hi is None else hi
    h = (w.upper[d] - w.lower[d]) / n
    return w.lower[d] + h * np.arange(lo, hi + 2, dtype=np.float64)


def level0_boxes(w: Workload):
    """Tile the level-0 domain with w.patch-sized boxes, x-major order.
    Returns a list of (lo, hi) inclusive index tuples."""
    ranges = []
    for d in range(w.ndim):
        n, p = w.ncells[d], w.patch[d]
        ranges.append([(a, min(a + p, n) - 1) for a in range(0, n, p)])
    boxes = []

    def rec(d, lo, hi):
        if d == w.ndim:
            boxes.append((tuple(lo), tuple(hi)))
            return
        for a, b in ranges[d]:
            rec(d + 1, lo + [a], hi + [b])
    rec(0, [], [])
    return boxes


# ---------------------------------------------------------------- profiles
def _Phi(z):
    """Standard normal CDF, written with erfc on the tail side for accuracy."""
    z = np.asarray(z, dtype=np.float64)
    return np.where(z < 0, 0.5 * special.erfc(-z / SQRT2), 1.0 - 0.5 * special.erfc(z / SQRT2))


def _normal_cell_mass(a, b, mu=0.0, sigma=1.0):
    """Integral over [a,b] of N(v; mu, sigma) with tail-accurate differences."""
    za = (np.asarray(a) - mu) / sigma
    zb = (np.asarray(b) - mu) / sigma
    upper = 0.5 * (special.erfc(za / SQRT2) - special.erfc(zb / SQRT2))     # good for z>0
    lower = 0.5 * (special.erfc(-zb / SQRT2) - special.erfc(-za / SQRT2))   # good for z<0
    return np.where(za >= 0, upper, np.where(zb <= 0, lower, _Phi(zb) - _Phi(za)))


def _v2_maxwellian_cell_mass(a, b):
    """Integral over [a,b] of v^2 exp(-v^2/2)/sqrt(2pi) = [Phi(v) - v phi(v)]_a^b."""
    phi = lambda v: np.exp(-0.5 * v * v) / math.sqrt(2 * math.pi)
    return _normal_cell_mass(a, b) - (b * phi(b) - a * phi(a))


def v_profile_cell_average(kind: str, edges: np.ndarray) -> np.ndarray:
    """Exact cell averages of the unperturbed 1D velocity profile on cells given by edges."""
    a, b = edges[:-1], edges[1:]
    h = b - a
    if kind in ("landau", "landau2d"):
        m = _normal_cell_mass(a, b)
    elif kind == "twostream":
        m = _v2_maxwellian_cell_mass(a, b)
    elif kind == "bump":  # BASELINE.json C4: 0.9 M(v;0,1) + 0.1 M(v;4.5,0.5)
        m = 0.9 * _normal_cell_mass(a, b, 0.0, 1.0) + 0.1 * _normal_cell_mass(a, b, 4.5, 0.5)
    else:
        raise ValueError(kind)
    return m / h


def _cos_cell_average(k: float, edges: np.ndarray) -> np.ndarray:
    """Cell averages of cos(k x)."""
    a, b = edges[:-1], edges[1:]
    return (np.sin(k * b) - np.sin(k * a)) / (k * (b - a))


def _sin_cell_average(k: float, edges: np.ndarray) -> np.ndarray:
    a, b = edges[:-1], edges[1:]
    return (np.cos(k * a) - np.cos(k * b)) / (k * (b - a))


def initial_cell_averages(w: Workload, ratio: Sequence[int] = None, box=None) -> np.ndarray:
    """Exact cell averages of f0 on the cells of ``box`` (inclusive (lo, hi), level
    index space at ``ratio`` to level 0; default the whole domain)."""
    ratio = tuple(ratio or (1,) * w.ndim)
    if box is None:
        box = (tuple(0 for _ in range(w.ndim)),
               tuple(w.ncells[d] * ratio[d] - 1 for d in range(w.ndim)))
    lo, hi = box
    e = [cell_edges(w, d, ratio[d], lo[d], hi[d]) for d in range(w.ndim)]
    if w.ncfg == 1:
        xs = 1.0 + w.alpha * _cos_cell_average(w.k[0], e[0])
        vs = v_profile_cell_average(w.ic, e[1])
        return np.ascontiguousarray(xs[:, None] * vs[None, :])
    # 2D+2V: M(vx) M(vy) (1 + alpha cos(kx x) cos(ky y))
    cx = _cos_cell_average(w.k[0], e[0])
    cy = _cos_cell_average(w.k[1], e[1])
    xy = 1.0 + w.alpha * cx[:, None] * cy[None, :]
    vx = v_profile_cell_average(w.ic, e[2])
    vy = v_profile_cell_average(w.ic, e[3])
    return np.ascontiguousarray(xy[:, :, None, None] * vx[None, None, :, None] * vy[None, None, None, :])


def background_profile(w: Workload, ratio: Sequence[int] = None, ghost: int = GHOST) -> np.ndarray:
    """Cell averages of the unperturbed velocity profile f0(v) over the level's whole
    velocity index range INCLUDING ``ghost`` cells on each side.
    1D+1V: shape (Nv + 2g,).  2D+2V: shape (Nvx + 2g, Nvy + 2g)."""
    ratio = tuple(ratio or (1,) * w.ndim)
    prof = []
    for d in range(w.ncfg, w.ndim):
        n = w.ncells[d] * ratio[d]
        prof.append(v_profile_cell_average(w.ic, cell_edges(w, d, ratio[d], -ghost, n - 1 + ghost)))
    if w.ncfg == 1:
        return np.ascontiguousarray(prof[0])
    return np.ascontiguousarray(prof[0][:, None] * prof[1][None, :])


def prescribed_field(w: Workload, ratio: Sequence[int] = None) -> np.ndarray:
    """C5: exact 2D cell averages of E = 0.1 (cos x, sin y).  Shape (2, Nx, Ny)."""
    assert w.field == "prescribed" and w.ncfg == 2
    ratio = tuple(ratio or (1,) * w.ndim)
    ex = 0.1 * _cos_cell_average(1.0, cell_edges(w, 0, ratio[0]))
    ey = 0.1 * _sin_cell_average(1.0, cell_edges(w, 1, ratio[1]))
    nx, ny = ex.size, ey.size
    return np.ascontiguousarray(np.stack([np.repeat(ex[:, None], ny, 1),
                                          np.repeat(ey[None, :], nx, 0)]))


def _profile_mass(w: Workload) -> float:
    return {"landau": 1.0, "landau2d": 1.0, "twostream": 1.0, "bump": 1.0}[w.ic]


def fixed_dt(w: Workload, ratio: Sequence[int] = None, cfl: float = 0.5) -> float:
    """Fixed time step (SURVEY.md 8(c) reading #17): cfl / sum_d(max|a_d|/h_d) with the
    cell-centre velocity bound for the x-advection and the continuum linear-field bound
    |E| <= alpha*mass/k (or the prescribed amplitude 0.1 for C5) for the v-advection.
    For AMR (C3) pass the finest ratio: spacing of the finest level, domain-wide bounds."""
    h = spacing(w, ratio)
    rate = 0.0
    for d in range(w.ncfg):
        vd = w.ncfg + d
        vmax = max(abs(w.lower[vd] + 0.5 * h[vd]), abs(w.upper[vd] - 0.5 * h[vd]))
        rate += vmax / h[d]
    for d in range(w.ncfg):
        vd = w.ncfg + d
        emax = 0.1 if w.field == "prescribed" else w.alpha * _profile_mass(w) / w.k[d]
        rate += emax / h[vd]
    return cfl / rate


# ---------------------------------------------------------------- random
def random_field(shape, seed: int, lo: float = -1.0, hi: float = 1.0) -> np.ndarray:
    rng = np.random.default_rng(seed)
    return rng.uniform(lo, hi, size=shape).astype(np.float64)


def random_positive_field(shape, seed: int) -> np.ndarray:
    """Positive, O(1) field with smooth structure plus noise (exercises upwind weights)."""
    rng = np.random.default_rng(seed)
    grids = np.meshgrid(*[np.linspace(0, 2 * np.pi, n, endpoint=False) for n in shape], indexing="ij")
    smooth = np.ones(shape)
    for g in grids:
        smooth = smooth + 0.3 * np.sin(g * rng.integers(1, 4) + rng.uniform(0, 6.28))
    return np.ascontiguousarray(smooth + 0.05 * rng.standard_normal(shape))
