"""Domain value types and host-side parameter selection for slab (quasi-2D) Coulomb systems.

The geometry is periodic in x and y and confined to ``0 <= z <= lz``; optional
uniformly charged planes sit at z = 0 and z = lz.  Units are reduced Gaussian
(bare pair potential ``q_i q_j / r``).

This module mirrors the value types of the reference package so that it is a
drop-in for the RBSE2D energy/force path:

* ``BoxGeometry``      -- reference ``pkg/src/slabewald/core.py:25-51``
* ``ParticleSystem``   -- ``core.py:54-84``
* ``make_system``      -- ``core.py:87-100`` (also accepts the box in the 4th
  positional slot, the call form used throughout the reference tests, e.g.
  ``tests/test_soewald2d.py:122``)
* ``EwaldParams``      -- ``core.py:103-120``
* ``enumerate_kmodes`` -- ``core.py:123-138``
* ``make_ewald_params``-- ``core.py:141-149``
* ``validate_neutrality`` -- ``core.py:152-163``
* ``choose_alpha``     -- ``core.py:211-232``
* ``sort_by_z``        -- ``core.py:203-208``; here it runs the device radix sort
  (bit-exact with the reference bucket sort, which equals a stable argsort).

Everything here is host-side setup (per run, not per step) except ``sort_by_z``.
"""

from __future__ import annotations

from dataclasses import dataclass, field
import math

import numpy as np

SQRT_PI = math.sqrt(math.pi)
NEUTRALITY_TOL = 1e-12


@dataclass(frozen=True)
class BoxGeometry:
    """Cell ``[0,lx) x [0,ly)`` periodic in-plane, ``[0,lz]`` confined in z.

    ``sigma_top`` / ``sigma_bot`` are surface charge densities of the planes at
    z = lz and z = 0 (reference ``core.py:25-51``).
    """

    lx: float
    ly: float
    lz: float
    sigma_top: float = 0.0
    sigma_bot: float = 0.0

    def __post_init__(self):
        if not (self.lx > 0 and self.ly > 0 and self.lz > 0):
            raise ValueError("box lengths must be positive")
        if not (math.isfinite(self.sigma_top) and math.isfinite(self.sigma_bot)):
            raise ValueError("slab charge densities must be finite")

    @property
    def area(self) -> float:
        return self.lx * self.ly

    @property
    def volume(self) -> float:
        return self.lx * self.ly * self.lz


@dataclass
class ParticleSystem:
    """Charges, masses, positions (N,3) and velocities (N,3), all float64 C-contiguous."""

    charge: np.ndarray
    mass: np.ndarray
    pos: np.ndarray
    vel: np.ndarray

    def __post_init__(self):
        as64 = lambda a: np.ascontiguousarray(a, dtype=np.float64)  # noqa: E731
        self.charge, self.mass = as64(self.charge), as64(self.mass)
        self.pos, self.vel = as64(self.pos), as64(self.vel)
        n = self.charge.shape[0]
        shapes_ok = (self.mass.shape == (n,) and self.pos.shape == (n, 3)
                     and self.vel.shape == (n, 3))
        if not shapes_ok:
            raise ValueError("inconsistent array shapes")
        if n and not bool(np.all(self.mass > 0)):
            raise ValueError("masses must be positive")

    @property
    def n(self) -> int:
        return int(self.charge.shape[0])

    def copy(self) -> "ParticleSystem":
        return ParticleSystem(self.charge.copy(), self.mass.copy(), self.pos.copy(),
                              self.vel.copy())


def make_system(charge, mass, pos, vel=None, box: BoxGeometry | None = None) -> ParticleSystem:
    """Build a ParticleSystem; with a box, wrap x,y into the cell and check z.

    The reference signature is ``make_system(charge, mass, pos, vel=None, box=None)``
    but its own tests pass the box as the 4th positional argument; a
    ``BoxGeometry`` found in the ``vel`` slot is therefore treated as the box.
    """
    if isinstance(vel, BoxGeometry):
        if box is not None:
            raise TypeError("box given twice")
        vel, box = None, vel
    pos = np.array(pos, dtype=np.float64).reshape(-1, 3)
    n = pos.shape[0]
    vel = np.zeros((n, 3)) if vel is None else np.asarray(vel, dtype=np.float64)
    if box is not None:
        pos[:, 0] = np.mod(pos[:, 0], box.lx)
        pos[:, 1] = np.mod(pos[:, 1], box.ly)
        if n and (pos[:, 2].min() < 0 or pos[:, 2].max() > box.lz):
            raise ValueError("z coordinates must lie in [0, lz]")
    return ParticleSystem(np.asarray(charge, dtype=np.float64),
                          np.asarray(mass, dtype=np.float64), pos, vel)


@dataclass(frozen=True)
class EwaldParams:
    """alpha, s, the coupled cutoffs r_c = s/alpha, k_c = 2 s alpha, and the
    (K,3) mode table of (kx, ky, |k|) (reference ``core.py:103-120``)."""

    alpha: float
    s: float
    r_c: float
    k_c: float
    kmodes: np.ndarray = field(repr=False)

    def __post_init__(self):
        if not (self.alpha > 0 and self.s > 0):
            raise ValueError("alpha and s must be positive")


def enumerate_kmodes(box: BoxGeometry, k_c: float) -> np.ndarray:
    """All nonzero lattice modes 2*pi*(mx/lx, my/ly) with |k| <= k_c.

    Order is lexicographic in (|k|, kx, ky) so equal-|k| rings are contiguous
    (reference ``core.py:123-138``; the ``1e-9`` / ``1e-12`` roundoff
    allowances are part of the contract).
    """
    step_x = 2.0 * np.pi / box.lx
    step_y = 2.0 * np.pi / box.ly
    nx = int(np.floor(k_c / step_x + 1e-9))
    ny = int(np.floor(k_c / step_y + 1e-9))
    ix = np.repeat(np.arange(-nx, nx + 1), 2 * ny + 1)
    iy = np.tile(np.arange(-ny, ny + 1), 2 * nx + 1)
    kx = step_x * ix
    ky = step_y * iy
    kn = np.hypot(kx, ky)
    sel = (kn > 0) & (kn <= k_c * (1 + 1e-12))
    kx, ky, kn = kx[sel], ky[sel], kn[sel]
    idx = np.lexsort((ky, kx, kn))
    return np.column_stack([kx[idx], ky[idx], kn[idx]])


def make_ewald_params(alpha: float, s: float, box: BoxGeometry) -> EwaldParams:
    if alpha <= 0.0:
        raise ValueError("alpha must be positive")
    if s <= 0.0:
        raise ValueError("s must be positive")
    k_c = 2.0 * s * alpha
    return EwaldParams(alpha=alpha, s=s, r_c=s / alpha, k_c=k_c,
                       kmodes=enumerate_kmodes(box, k_c))


def validate_neutrality(system: ParticleSystem, box: BoxGeometry,
                        tol: float = NEUTRALITY_TOL) -> tuple[bool, float]:
    """(ok, |sum q + (sigma_top + sigma_bot) A|) with a tolerance relative to sum|q|."""
    resid = float(abs(system.charge.sum() + (box.sigma_top + box.sigma_bot) * box.area))
    scale = max(1.0, float(np.abs(system.charge).sum()))
    return resid <= tol * scale, resid


def choose_alpha(n: int, box: BoxGeometry, mode: str = "balanced",
                 prefactor: float = 1.0, s: float = 4.0) -> float:
    """Splitting parameter from the cost-balance laws (reference ``core.py:211-232``).

    ``linear``: alpha = prefactor (N/V)^(1/3) (fixed short-range cost per
    particle; what the random-batch solver uses).  ``balanced``: alpha ~
    N^(1/5) / (lx^(2/5) ly^(2/5) lz^(1/5)), switching to N^(1/4)/sqrt(lx ly)
    when s/alpha would exceed lz.
    """
    if n < 1:
        raise ValueError("need at least one particle")
    if mode == "linear":
        return prefactor * (n / box.volume) ** (1.0 / 3.0)
    if mode == "balanced":
        a = prefactor * n ** 0.2 / (box.lx ** 0.4 * box.ly ** 0.4 * box.lz ** 0.2)
        if s / a > box.lz:
            a = prefactor * n ** 0.25 / np.sqrt(box.lx * box.ly)
        return a
    raise ValueError(f"unknown alpha mode: {mode!r}")


def sort_by_z(system: ParticleSystem, lz: float) -> np.ndarray:
    """Stable permutation ordering particles by ascending z (int64, input indices).

    Runs the device LSD radix sort (``slab_sort_by_z`` in the C-ABI).  Bit-exact
    with the reference bucket sort (``core.py:166-208``), which equals
    ``np.argsort(z, kind="stable")``; ``-0.0`` ties with ``+0.0``.
    """
    z = system.pos[:, 2]
    if not np.all(np.isfinite(z)):
        raise ValueError("z coordinates must be finite")
    from .engine import device_sort_perm
    return device_sort_perm(np.ascontiguousarray(z), float(lz))


# ---------------------------------------------------------------------------
# particle CSV (reference core.py:305-329): header id,q,m,x,y,z,vx,vy,vz, rows in
# any order, read back ordered by id; written with 17 significant digits so a
# save / load round trip is exact.
# ---------------------------------------------------------------------------
PARTICLE_CSV_HEADER = "id,q,m,x,y,z,vx,vy,vz"


def load_particles(path, box: BoxGeometry | None = None) -> ParticleSystem:
    import csv
    with open(path, newline="") as fh:
        rows = list(csv.reader(fh))
    if not rows or [c.strip() for c in rows[0]] != PARTICLE_CSV_HEADER.split(","):
        raise ValueError(f"particle CSV must have header {PARTICLE_CSV_HEADER}")
    body = [r for r in rows[1:] if r and any(c.strip() for c in r)]
    a = np.array([[float(c) for c in r] for r in body], dtype=np.float64).reshape(-1, 9)
    a = a[np.argsort(a[:, 0], kind="stable")]
    return make_system(a[:, 1], a[:, 2], a[:, 3:6], a[:, 6:9], box=box)


def save_particles(path, system: ParticleSystem) -> None:
    vel = system.vel if system.vel is not None else np.zeros((system.n, 3))
    lines = [PARTICLE_CSV_HEADER]
    for i in range(system.n):
        vals = (system.charge[i], system.mass[i], *system.pos[i], *vel[i])
        lines.append(str(i) + "," + ",".join(f"{v:.17g}" for v in vals))
    with open(path, "w") as fh:
        fh.write("\n".join(lines) + "\n")
