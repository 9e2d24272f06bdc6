"""Multi-GPU work split for one evaluation; host-side, no device code.

Particles are replicated on every rank.  Rank r of W evaluates
  * the sampled modes [mode_slice(P, r, W)]      (every (mode, SOE pair, direction)
    chain is independent once the particles are z-sorted),
  * the short-range home particles [home_range(n, r, W)] of the stable cell
    order (``slab_evaluate`` applies the same formula on device),
  * and, on the lead rank only, the k = 0 mode, the constants (C_Q / u_q, self,
    slab planes) and the plane forces.
Summing the per-rank (forces, energies) -- ONE all-reduce of a packed buffer --
gives the single-GPU result up to summation order.
"""

from __future__ import annotations


def mode_slice(P: int, rank: int, world: int) -> tuple[int, int]:
    return P * rank // world, P * (rank + 1) // world


def home_range(n: int, rank: int, world: int) -> tuple[int, int]:
    return n * rank // world, n * (rank + 1) // world


def is_lead(rank: int) -> bool:
    return rank == 0
