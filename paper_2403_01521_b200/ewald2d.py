"""Short-range, self and slab-plane terms; the EnergyBreakdown record.

Reference ``pkg/src/slabewald/ewald2d.py``:
  * ``EnergyBreakdown`` 36-48 (total = u_s + u_l_k + u_l_0 - u_self + u_ps)
  * ``short_range_energy_forces`` 280-303 -> device cell-list kernel
    (``slab_short_range``; cell rules of build_cell_list 141-157, pair kernels
    160-277)
  * ``self_energy`` 527-529, ``slab_energy_forces`` 532-545: O(N) numpy
    formulas here exactly as in the reference (on the evaluation path the same
    terms are computed on device by ``assemble_energy_kernel``).

The O(N^2 K) Ewald2D reference solver (``fourier_energy_forces_ref``,
``zero_mode_energy_forces_ref``, ``ref_energy_forces``, ``total_energy_ref``,
ewald2d.py:310-574) runs on device as the accuracy oracle of SURVEY 8(f) rank 4
(``ewald_ref.cu``); the brute-force lattice-sum oracle and the error predictors
stay out of scope.
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


def status_of(energy, summed: bool = False) -> int:
    """Status bits from an evaluation's energy vector; ``summed``: the vector went
    through the multi-GPU SUM all-reduce (decode slot 7's 8-bit-per-bit counters)."""
    if not summed:
        return int(energy[5])
    v = int(round(float(energy[7])))
    st = 0
    for k in range(6):
        if (v >> (8 * k)) & 255:
            st |= 1 << k
    return st


def raise_on_status(status: int) -> None:
    from ._native import SLAB_STATUS_COINCIDENT, SLAB_STATUS_NONFINITE
    if status & SLAB_STATUS_NONFINITE:  # checked first, like sort_by_z (core.py:206-207)
        raise ValueError("z coordinates must be finite")
    if status & SLAB_STATUS_COINCIDENT:
        raise ValueError("coincident particles: short-range energy is singular")


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


# ---------------------------------------------------------------------------
# O(N^2 K) Ewald2D reference solver on device (ewald2d.py:310-574)
# ---------------------------------------------------------------------------
def _ring_table(params, box: BoxGeometry):
    """Integer (mx, my) per mode, ring id per mode and the ring norms: modes of
    equal |k| (to 1e-12 relative, in the sorted mode order) share the xi kernels
    (ewald2d.py:310-328)."""
    km = params.kmodes
    mx = np.rint(km[:, 0] * box.lx / (2 * np.pi)).astype(np.int32)
    my = np.rint(km[:, 1] * box.ly / (2 * np.pi)).astype(np.int32)
    ring = np.zeros(len(km), dtype=np.int32)
    kap = [km[0, 2]] if len(km) else []
    for t in range(1, len(km)):
        if km[t, 2] - kap[-1] > 1e-12 * max(1.0, kap[-1]):
            kap.append(km[t, 2])
        ring[t] = len(kap) - 1
    return mx, my, ring, np.array(kap, dtype=np.float64)


def fourier_energy_forces_ref(system: ParticleSystem, box: BoxGeometry, params,
                              variant: str = "stable"):
    """Nonzero-mode Fourier energy (pair sum + the force-free charge term u_q) and
    forces by direct pairwise summation over the mode set, on device."""
    from scipy.special import erfc as _erfc
    n = system.n
    if params.kmodes.shape[0] == 0:
        return 0.0, np.zeros((n, 3))
    if variant not in ("stable", "naive"):
        raise ValueError(f"unknown variant {variant!r}")
    Q = float(np.sum(system.charge ** 2))
    kn = params.kmodes[:, 2]
    u_q = float(np.sum(np.pi * Q / (kn * box.area) * _erfc(kn / (2 * params.alpha))))
    if n < 2:
        return u_q, np.zeros((n, 3))
    from .engine import get_engine, host_result, to_device
    import torch
    from ._native import check
    eng = get_engine()
    mx, my, ring, kap = _ring_table(params, box)
    mxy = torch.as_tensor(np.ascontiguousarray(np.column_stack([mx, my]))).to(eng.device)
    ring_t = torch.as_tensor(ring).to(eng.device)
    kap_t = to_device(kap)
    pos, q = to_device(system.pos), to_device(system.charge)
    forces = torch.empty((n, 3), dtype=torch.float64, device=eng.device)
    energy = torch.zeros(8, dtype=torch.float64, device=eng.device)
    import ctypes
    p = lambda t: ctypes.c_void_p(t.data_ptr())
    check(eng.lib.slab_ewald_ref_fourier(
        eng.ctx, p(pos), p(q), n, float(box.lx), float(box.ly), float(params.alpha), p(mxy),
        p(ring_t), len(ring), p(kap_t), len(kap), int(np.max(np.abs(mx))),
        int(np.max(np.abs(my))), 1 if variant == "naive" else 0, p(forces), p(energy),
        eng._stream()), "slab_ewald_ref_fourier")
    e, f = host_result(energy, forces)
    return float(e[0]) + u_q, f


def fourier_energy_ref(system: ParticleSystem, box: BoxGeometry, params,
                       variant: str = "stable") -> float:
    u, _ = fourier_energy_forces_ref(system, box, params, variant)
    return u


def zero_mode_energy_forces_ref(system: ParticleSystem, box: BoxGeometry, alpha: float):
    """k = 0 mode energy (ordered pairs including i = j) and its z-forces, direct
    pairwise sum on device (ewald2d.py:477-519)."""
    n = system.n
    Q = float(np.sum(system.charge ** 2))
    const = -SQRT_PI * Q / (alpha * box.area)
    if n < 2:
        return (const if n else 0.0), np.zeros((n, 3))
    from .engine import get_engine, host_result, to_device
    import ctypes
    import torch
    from ._native import check
    eng = get_engine()
    pos, q = to_device(system.pos), to_device(system.charge)
    fz = torch.empty(n, dtype=torch.float64, device=eng.device)
    energy = torch.zeros(8, dtype=torch.float64, device=eng.device)
    p = lambda t: ctypes.c_void_p(t.data_ptr())
    check(eng.lib.slab_ewald_ref_zero(eng.ctx, p(pos), p(q), n, float(alpha), p(fz), p(energy),
                                      eng._stream()), "slab_ewald_ref_zero")
    e, fzh = host_result(energy, fz)
    pref = 2.0 * np.pi / box.area
    forces = np.zeros((n, 3))
    forces[:, 2] = pref * fzh
    return float(-pref * e[0] + const), forces


def zero_mode_energy_ref(system: ParticleSystem, box: BoxGeometry, alpha: float) -> float:
    u, _ = zero_mode_energy_forces_ref(system, box, alpha)
    return u


class Ewald2DDevice:
    """The O(N^2 K) Ewald2D evaluation (ewald2d.py:548-561) enqueued into caller
    device buffers with no host synchronisation: the force field of an MD run
    with ``solver="ewald2d"`` (reference md.py:149-150).  Per-run constants (the
    ring table of the mode set, u_q, the k = 0 constant) are prepared once."""

    def __init__(self, eng, params, box: BoxGeometry, Q: float, variant: str = "stable"):
        from scipy.special import erfc as _erfc
        import torch
        from .engine import to_device
        self.eng, self.params, self.box = eng, params, box
        self.variant = 1 if variant == "naive" else 0
        km = params.kmodes
        self.nmode = km.shape[0]
        self.u_q = float(np.sum(np.pi * Q / (km[:, 2] * box.area) *
                                _erfc(km[:, 2] / (2 * params.alpha)))) if self.nmode else 0.0
        self.const0 = -SQRT_PI * Q / (params.alpha * box.area)
        if self.nmode:
            mx, my, ring, kap = _ring_table(params, box)
            self.mxy = torch.as_tensor(np.ascontiguousarray(np.column_stack([mx, my]))).to(
                eng.device)
            self.ring = torch.as_tensor(ring).to(eng.device)
            self.kap = to_device(kap)
            self.nring, self.mxmax, self.mymax = len(kap), int(np.max(np.abs(mx))), int(
                np.max(np.abs(my)))

    def enqueue(self, pos, q, forces, energy, status):
        """forces (N,3) = total Ewald2D forces; energy[0:5] = (u_s, u_l_k, u_l_0,
        u_self, u_ps), energy[5] = status bits (also OR-ed into ``status``)."""
        import ctypes
        import torch
        from ._native import SlabBox, check
        eng, box, prm = self.eng, self.box, self.params
        n = q.numel()
        dev = eng.device
        p = lambda t: ctypes.c_void_p(t.data_ptr())
        sbox = SlabBox(box.lx, box.ly, box.lz, box.sigma_top, box.sigma_bot)
        st = eng._stream()
        es = torch.zeros(1, dtype=torch.float64, device=dev)
        sr_status = torch.zeros(1, dtype=torch.int32, device=dev)
        check(eng.lib.slab_short_range(eng.ctx, p(pos), p(q), n, sbox, float(prm.alpha),
                                       float(prm.r_c), p(forces), p(es), p(sr_status), st),
              "slab_short_range")
        ek = torch.zeros(8, dtype=torch.float64, device=dev)
        if self.nmode and n >= 2:
            fk = torch.empty((n, 3), dtype=torch.float64, device=dev)
            check(eng.lib.slab_ewald_ref_fourier(
                eng.ctx, p(pos), p(q), n, float(box.lx), float(box.ly), float(prm.alpha),
                p(self.mxy), p(self.ring), self.nmode, p(self.kap), self.nring, self.mxmax,
                self.mymax, self.variant, p(fk), p(ek), st), "slab_ewald_ref_fourier")
            forces += fk
        e0 = torch.zeros(8, dtype=torch.float64, device=dev)
        if n >= 2:
            fz = torch.empty(n, dtype=torch.float64, device=dev)
            check(eng.lib.slab_ewald_ref_zero(eng.ctx, p(pos), p(q), n, float(prm.alpha), p(fz),
                                              p(e0), st), "slab_ewald_ref_zero")
            forces[:, 2] += (2.0 * np.pi / box.area) * fz
        ec = eng.constant_terms(pos, q, box, prm.alpha)
        forces[:, 2] += (-2.0 * np.pi * (box.sigma_top - box.sigma_bot)) * q
        energy[0] = es[0]
        energy[1] = ek[0] + self.u_q
        energy[2] = -(2.0 * np.pi / box.area) * e0[0] + (self.const0 if n else 0.0)
        energy[3] = ec[3]
        energy[4] = ec[4]
        energy[5] = sr_status[0].to(torch.float64)
        status.bitwise_or_(sr_status)


def ref_energy_forces(system: ParticleSystem, box: BoxGeometry, params,
                      variant: str = "stable"):
    """Full Ewald2D reference evaluation: EnergyBreakdown plus forces
    (ewald2d.py:548-562), with the reference's neutrality check."""
    from .core import validate_neutrality
    ok, residual = validate_neutrality(system, box)
    if not ok:
        raise ValueError(f"system is not charge neutral (residual {residual:g})")
    u_s, f_s = short_range_energy_forces(system, box, params.alpha, params.r_c)
    u_k, f_k = fourier_energy_forces_ref(system, box, params, variant)
    u_0, f_0 = zero_mode_energy_forces_ref(system, box, params.alpha)
    _, f_ps = slab_energy_forces(system, box)
    # u_self and u_ps from the same device reduction as the SOE / RB assembly, so
    # every solver reports the shared terms bitwise alike (reference
    # test_total_breakdown_shares_short_range_and_slab_with_reference)
    from .engine import get_engine, to_device
    eng = get_engine()
    e = eng.constant_terms(to_device(system.pos), to_device(system.charge), box,
                           params.alpha).cpu().numpy()
    u_self, u_ps = float(e[3]), float(e[4])
    return (EnergyBreakdown(u_s=u_s, u_l_k=u_k, u_l_0=u_0, u_self=u_self, u_ps=u_ps),
            f_s + f_k + f_0 + f_ps)


def total_energy_ref(system: ParticleSystem, box: BoxGeometry, params,
                     variant: str = "stable") -> EnergyBreakdown:
    bd, _ = ref_energy_forces(system, box, params, variant)
    return bd
