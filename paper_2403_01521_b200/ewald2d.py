"""Short-range, self and slab-plane terms; the EnergyBreakdown record.

Reference ``pkg/src/slabewald/ewald2d.py``:
  * ``EnergyBreakdown`` 36-48 (total = u_s + u_l_k + u_l_0 - u_self + u_ps)
  * ``short_range_energy_forces`` 280-303 -> device cell-list kernel
    (``slab_short_range``; cell rules of build_cell_list 141-157, pair kernels
    160-277)
  * ``self_energy`` 527-529, ``slab_energy_forces`` 532-545: O(N) numpy
    formulas here exactly as in the reference (on the evaluation path the same
    terms are computed on device by ``assemble_energy_kernel``).

The O(N^2 K) Ewald2D reference solver and the lattice-sum oracle of the
reference module are accuracy oracles outside this hot path.
"""

from __future__ import annotations

from dataclasses import dataclass
import math

import numpy as np

from .core import BoxGeometry, ParticleSystem

SQRT_PI = math.sqrt(math.pi)


@dataclass(frozen=True)
class EnergyBreakdown:
    """Energy parts; total = u_s + u_l_k + u_l_0 - u_self + u_ps."""

    u_s: float
    u_l_k: float
    u_l_0: float
    u_self: float
    u_ps: float

    @property
    def total(self) -> float:
        return self.u_s + self.u_l_k + self.u_l_0 - self.u_self + self.u_ps


def check_short_range_cutoff(box: BoxGeometry, r_c: float) -> None:
    if r_c > min(box.lx, box.ly) / 2 + 1e-12:
        raise ValueError("r_c must not exceed half the in-plane box size")


def raise_on_status(status: int) -> None:
    from ._native import SLAB_STATUS_COINCIDENT, SLAB_STATUS_NONFINITE, SLAB_STATUS_SINGULAR
    if status & SLAB_STATUS_NONFINITE:  # checked first, like sort_by_z (core.py:206-207)
        raise ValueError("z coordinates must be finite")
    if status & SLAB_STATUS_COINCIDENT:
        raise ValueError("coincident particles: short-range energy is singular")
    if status & SLAB_STATUS_SINGULAR:
        raise NotImplementedError(
            "an SOE exponent alpha*s_l lies within 2e-6 k of a sampled |k|: the analytic-limit "
            "branch of soewald2d.py:116-124 is not implemented on device")


def short_range_energy_forces(system: ParticleSystem, box: BoxGeometry, alpha: float,
                              r_c: float):
    """Minimum-image erfc pair sum within r_c, on device.  Returns (u_s, forces)."""
    check_short_range_cutoff(box, r_c)
    n = system.n
    if n < 2:
        return 0.0, np.zeros((n, 3))
    from .engine import get_engine, to_device
    eng = get_engine()
    pos = to_device(system.pos)
    q = to_device(system.charge)
    energy, forces, status = eng.short_range(pos, q, box, alpha, r_c)
    st = int(status.cpu().item())
    raise_on_status(st)
    return float(energy.cpu().item()), forces.cpu().numpy()


def self_energy(system: ParticleSystem, alpha: float) -> float:
    """Gaussian self interaction (alpha/sqrt(pi)) sum q_i^2 (reference 527-529)."""
    return float(alpha / SQRT_PI * np.sum(system.charge ** 2))


def slab_energy_forces(system: ParticleSystem, box: BoxGeometry):
    """Charged-plane term: phi(z) = -2 pi [sigma_top (lz - z) + sigma_bot z] (532-545)."""
    z = system.pos[:, 2]
    phi = -2.0 * np.pi * (box.sigma_top * (box.lz - z) + box.sigma_bot * z)
    u = float(np.dot(system.charge, phi))
    forces = np.zeros((system.n, 3))
    forces[:, 2] = -2.0 * np.pi * system.charge * (box.sigma_top - box.sigma_bot)
    return u, forces
