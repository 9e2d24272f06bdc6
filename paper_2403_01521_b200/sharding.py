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


# Modes are split evenly: a rank's sweep cost is quantised by whole warps of
# items, so trimming the lead rank's modes buys little (LEAD_MODE_DISCOUNT = 0);
# the lead's extra k = 0 mode work is balanced on the short range instead.
LEAD_MODE_DISCOUNT = 0


def mode_slice(P: int, rank: int, world: int) -> tuple[int, int]:
    """Contiguous mode range of rank r: equal shares of P + d "mode units", the
    lead rank's share reduced by d (its k = 0 mode work)."""
    if world <= 1:
        return 0, P
    d = min(LEAD_MODE_DISCOUNT, P // world)

    def bound(r):
        if r <= 0:
            return 0
        if r >= world:
            return P
        return min(P, max(0, (P + d) * r // world - d))
    return bound(rank), bound(rank + 1)


# The lead rank takes a reduced share of the short-range home particles: it also
# runs the k = 0 mode and the assembly constants (~0.35 ms at cfg4, against a
# short-range share of ~3.5 ms / W).  Lead share in tenths of a regular share,
# measured on one B200 per rank count (tools/shard_step.py, z-split); slab_evaluate
# uses the same table (capi.cu home_bound).
LEAD_HOME_TENTHS = (10, 10, 8, 8, 7, 5, 4, 2, 1)  # index = world size, 0 beyond


def lead_home_tenths(world: int) -> int:
    return LEAD_HOME_TENTHS[world] if world < len(LEAD_HOME_TENTHS) else 0


def home_range(n: int, rank: int, world: int) -> tuple[int, int]:
    if world <= 1:
        return 0, n
    lead = lead_home_tenths(world)
    units = lead + 10 * (world - 1)

    def bound(r):
        if r <= 0:
            return 0
        if r >= world:
            return n
        return n * (lead + 10 * (r - 1)) // units
    return bound(rank), bound(rank + 1)


def is_lead(rank: int) -> bool:
    return rank == 0
