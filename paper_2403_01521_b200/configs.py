"""Seeded synthetic workloads for the five BASELINE.json configurations.

SURVEY.md section 8(d) fixes the shapes: charges listed cations first then
anions (as the reference CLI generator, ``pkg/src/slabewald/cli.py:225-260``),
masses 1, sigma_top = sigma_bot = 0, SOE from ``build_soe_contour(M)``, s = 4 and
alpha = choose_alpha(N, box, "linear") for the random-batch configs.  There is
no public dataset; these generators ARE the inputs (same numpy version on the
GPU box, so they regenerate bit-identically there).

``name`` -> Workload:
  cfg1      N=1000, 20^3 box, alpha=0.5, s=5 (r_c=10, k_c=5), full mode set, M=16
  cfg2      N=1e4, Lx=Ly=L, Lz=L/2 at density 0.1, RB P=100, M=16
  cfg3      N=1e5 thin slab Lz=0.1 Lx, exponential wall layers, RB P=200, M=24
  cfg4      N=999,999 2:1 electrolyte (+2/-1), Lx=Ly=2Lz, density 0.1, RB P=100, M=16
  cfg5_<N>  cube at density 0.1, N in {1e4,1e5,1e6,1e7}, RB P=100, M=16
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from .core import BoxGeometry, choose_alpha, make_ewald_params, make_system

DENSITY = 0.1

DESCRIPTIONS = {
    "cfg1": "N=1000 +-1 charges in a 20^3 box, alpha=0.5, r_c=10, full mode set (k <= k_c)",
    "cfg2": "N=1e4 neutral +-1 charges, Lx=Ly=L, Lz=L/2, density 0.1, RB",
    "cfg3": "N=1e5 +-1 charges, thin slab Lz=0.1 Lx, exponential wall layers (0.05 Lz), RB",
    "cfg4": "N=999999 2:1 electrolyte, Lx=Ly=2Lz, density 0.1, RB",
    "cfg5": "neutral +-1 charges in a cube at density 0.1, RB (throughput sweep)",
}


def describe(name: str) -> str:
    """One-line recipe of a workload (bench.py's config.workload)."""
    return DESCRIPTIONS.get(name.split("_")[0], name)


@dataclass
class Workload:
    name: str
    system: object
    box: BoxGeometry
    alpha: float
    s: float
    m: int
    P: int | None          # None = full deterministic mode sum (soe_energy_forces)
    seed: int

    @property
    def n(self) -> int:
        return self.system.n

    def params(self):
        return make_ewald_params(self.alpha, self.s, self.box)


def _pm_charges(n_pos: int, n_neg: int, q_pos: float = 1.0, q_neg: float = -1.0):
    return np.concatenate([np.full(n_pos, q_pos), np.full(n_neg, q_neg)])


def _uniform(rng, n, box):
    return rng.random((n, 3)) * np.array([box.lx, box.ly, box.lz])


def make_workload(name: str) -> Workload:
    if name == "cfg1":
        n, box, seed = 1000, BoxGeometry(20.0, 20.0, 20.0), 1
        rng = np.random.default_rng(seed)
        pos = _uniform(rng, n, box)
        q = _pm_charges(500, 500)
        return Workload(name, make_system(q, np.ones(n), pos, box=box), box, 0.5, 5.0, 16,
                        None, seed)
    if name == "cfg2":
        n, seed = 10_000, 2
        L = (2 * n / DENSITY) ** (1.0 / 3.0)
        box = BoxGeometry(L, L, L / 2)
        rng = np.random.default_rng(seed)
        pos = _uniform(rng, n, box)
        q = _pm_charges(n // 2, n // 2)
        return _rb(name, q, pos, box, 16, 100, seed)
    if name == "cfg3":
        n, seed = 100_000, 3
        L = (n / (0.1 * DENSITY)) ** (1.0 / 3.0)
        box = BoxGeometry(L, L, 0.1 * L)
        rng = np.random.default_rng(seed)
        xy = rng.random((n, 2)) * np.array([box.lx, box.ly])
        scale = 0.05 * box.lz
        d = rng.exponential(scale, size=n)
        bad = d > box.lz / 2
        while np.any(bad):
            d[bad] = rng.exponential(scale, size=int(bad.sum()))
            bad = d > box.lz / 2
        top = rng.random(n) < 0.5
        z = np.where(top, box.lz - d, d)
        pos = np.column_stack([xy, z])
        q = _pm_charges(n // 2, n // 2)
        return _rb(name, q, pos, box, 24, 200, seed)
    if name == "cfg4":
        n, seed = 999_999, 4
        lz = (n / (4 * DENSITY)) ** (1.0 / 3.0)
        box = BoxGeometry(2 * lz, 2 * lz, lz)
        rng = np.random.default_rng(seed)
        pos = _uniform(rng, n, box)
        q = _pm_charges(n // 3, 2 * n // 3, 2.0, -1.0)
        return _rb(name, q, pos, box, 16, 100, seed)
    if name.startswith("cfg5_"):
        n, seed = int(float(name.split("_", 1)[1])), 5
        L = (n / DENSITY) ** (1.0 / 3.0)
        box = BoxGeometry(L, L, L)
        rng = np.random.default_rng(seed)
        pos = _uniform(rng, n, box)
        q = _pm_charges(n // 2, n - n // 2)
        return _rb(name, q, pos, box, 16, 100, seed)
    if name.startswith("small_"):
        # small RB slab used by fast parity tests: small_<N>
        n, seed = int(name.split("_", 1)[1]), 7
        L = (2 * n / DENSITY) ** (1.0 / 3.0)
        box = BoxGeometry(L, L, L / 2)
        rng = np.random.default_rng(seed)
        pos = _uniform(rng, n, box)
        q = _pm_charges(n // 2, n - n // 2)
        return _rb(name, q, pos, box, 16, 24, seed)
    raise ValueError(f"unknown workload {name!r}")


def _rb(name, q, pos, box, m, P, seed) -> Workload:
    n = len(q)
    system = make_system(q, np.ones(n), pos, box=box)
    alpha = choose_alpha(n, box, "linear", prefactor=1.0, s=4.0)
    return Workload(name, system, box, alpha, 4.0, m, P, seed)
