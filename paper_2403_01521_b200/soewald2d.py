"""SOEwald2D on device: the deterministic full-mode solver and its part-wise entry points.

Drop-in for reference ``pkg/src/slabewald/soewald2d.py``:
  * ``recursive_pair_sum`` 42-64           -> ``slab_recursive_pair_sum``
  * ``fourier_energy_soe`` 304-332         -> ``slab_fourier_sweep`` / ``slab_evaluate``
  * ``fourier_mode_energy_soe`` 335-344
  * ``zero_mode_energy_soe`` 347-366       -> ``slab_zero_mode_sweep``
  * ``forces_soe`` 369-395, ``soe_energy_forces`` 398-438,
    ``total_energy_soe`` 441-452          -> ``slab_evaluate``
Same signatures, return types and error messages.  All sweeps, sorting and
assembly run in the CUDA library; host code only validates inputs and forms
the per-run constants (mode prefactors, u_q).
"""

from __future__ import annotations

import math

import numpy as np
from scipy.special import erfc

from .core import BoxGeometry, EwaldParams, ParticleSystem
from .ewald2d import (EnergyBreakdown, check_short_range_cutoff, raise_on_status)
from .soe import SOEApprox

SQRT_PI = math.sqrt(math.pi)
TWO_OVER_SQRT_PI = 2.0 / SQRT_PI


def full_sum_constants(params: EwaldParams, box: BoxGeometry, Q: float):
    """(commonv per mode, u_q) of the deterministic mode sum (soewald2d.py:408-422)."""
    kn = params.kmodes[:, 2]
    if kn.shape[0] == 0:
        return np.zeros(0), 0.0
    uq = float(np.sum(np.pi * Q / (kn * box.area) * erfc(kn / (2 * params.alpha))))
    cv = TWO_OVER_SQRT_PI * params.alpha * np.exp(-kn ** 2 / (4 * params.alpha ** 2))
    return np.ascontiguousarray(cv), uq


def _check_finite_z(system: ParticleSystem):
    if not np.all(np.isfinite(system.pos[:, 2])):
        raise ValueError("z coordinates must be finite")


def _check_sorted(z):
    if np.any(np.diff(np.asarray(z)) < 0):
        raise ValueError("recursion sweeps require z sorted ascending")


def device_evaluate(system: ParticleSystem, box: BoxGeometry, alpha: float, r_c: float,
                    soe: SOEApprox, modes, commonv, charge_const: float, want_forces=True,
                    skip_short_range=False):
    """One ``slab_evaluate_host`` call on the host arrays (uploads, evaluation and
    result download in one C call, one synchronisation); ``modes`` is a host
    (P,3) array or a device tensor (the device sampler's batch).  Returns
    (energy[8], forces or None)."""
    import torch

    from .engine import get_engine, to_device
    if not skip_short_range:
        check_short_range_cutoff(box, r_c)
    eng = get_engine()
    if torch.is_tensor(modes):
        mt = modes if modes.shape[0] else None
    else:
        modes = np.asarray(modes, dtype=np.float64).reshape(-1, 3)
        mt = to_device(modes) if modes.shape[0] else None
    cv = to_device(commonv) if isinstance(commonv, np.ndarray) else float(commonv)
    while True:
        e, f = eng.evaluate_host(system.pos, system.charge, box, alpha, r_c, soe, mt, cv,
                                 charge_const, want_forces=want_forces,
                                 skip_short_range=skip_short_range)
        if not eng.handle_overflow(int(e[5])):
            break
    raise_on_status(int(e[5]))  # includes the non-finite-z check done on device
    return e, f


def _breakdown(e) -> EnergyBreakdown:
    return EnergyBreakdown(u_s=float(e[0]), u_l_k=float(e[1]), u_l_0=float(e[2]),
                           u_self=float(e[3]), u_ps=float(e[4]))


def recursive_pair_sum(charge: np.ndarray, theta: np.ndarray, z: np.ndarray,
                       beta: complex) -> np.ndarray:
    """Forward recursion A_a = sum_{j<a} q_j exp(-i theta_j - beta (z_a - z_j)) on device."""
    z = np.asarray(z, dtype=np.float64)
    if np.any(np.diff(z) < 0):
        raise ValueError("z must be sorted ascending")
    beta = complex(beta)
    if beta.real < 0:
        raise ValueError("Re(beta) must be nonnegative")
    n = len(z)
    if n == 0:
        return np.zeros(0, dtype=np.complex128)
    from .engine import get_engine, to_device
    eng = get_engine()
    out = eng.recursive_pair_sum(to_device(charge), to_device(theta), to_device(z), beta)
    o = out.cpu().numpy()
    return o[:, 0] + 1j * o[:, 1]


def fourier_energy_soe(system: ParticleSystem, box: BoxGeometry, params: EwaldParams,
                       soe: SOEApprox, _presorted=None) -> float:
    """Energy of all nonzero modes (sweep + u_q) -- reference soewald2d.py:304-332."""
    kmodes = params.kmodes
    if _presorted is not None:
        x, y, z, q = (np.ascontiguousarray(a, dtype=np.float64) for a in _presorted)
        _check_sorted(z)
        Q = float(np.sum(q ** 2))
    else:
        _check_finite_z(system)
        Q = float(np.sum(system.charge ** 2))
    cv, uq = full_sum_constants(params, box, Q)
    n = len(_presorted[2]) if _presorted is not None else system.n
    if kmodes.shape[0] == 0 or n < 2:
        return uq
    if _presorted is None:
        e, _ = device_evaluate(system, box, params.alpha, params.r_c, soe, kmodes, cv, uq,
                               want_forces=False, skip_short_range=True)
        return float(e[1])
    from .engine import get_engine, to_device
    eng = get_engine()
    energy, status = eng.fourier_sweep(to_device(x), to_device(y), to_device(z), to_device(q),
                                       to_device(kmodes), to_device(cv), soe, params.alpha,
                                       box.area, want_forces=False)
    raise_on_status(int(status.cpu().item()))
    return float(energy.cpu().item()) + uq


def fourier_mode_energy_soe(system: ParticleSystem, box: BoxGeometry, params: EwaldParams,
                            soe: SOEApprox, mode_index: int) -> float:
    """Energy of a single nonzero mode including its charge term (335-344)."""
    kmodes = params.kmodes
    if not 0 <= mode_index < kmodes.shape[0]:
        raise IndexError("mode index out of range")
    sub = EwaldParams(alpha=params.alpha, s=params.s, r_c=params.r_c, k_c=params.k_c,
                      kmodes=kmodes[mode_index:mode_index + 1])
    return fourier_energy_soe(system, box, sub, soe)


def zero_mode_energy_soe(system: ParticleSystem, box: BoxGeometry, alpha: float,
                         soe: SOEApprox, _presorted=None) -> float:
    """k = 0 mode energy (347-366): -(2 pi/A) u_pair - sqrt(pi) Q/(alpha A)."""
    if _presorted is None:
        _check_finite_z(system)
        q_in = system.charge
    else:
        _, _, z, q = (np.ascontiguousarray(a, dtype=np.float64) for a in _presorted)
        _check_sorted(z)
        q_in = q
    n = len(q_in)
    Q = float(np.sum(np.asarray(q_in) ** 2))
    const = -SQRT_PI * Q / (alpha * box.area)
    if n < 2:
        return const if n else 0.0
    if _presorted is None:
        e, _ = device_evaluate(system, box, alpha, 1.0, soe, np.zeros((0, 3)), 0.0, 0.0,
                               want_forces=False, skip_short_range=True)
        return float(e[2])
    from .engine import get_engine, to_device
    eng = get_engine()
    up = eng.zero_mode_sweep(to_device(z), to_device(q), soe, alpha, want_forces=False)
    return float(-2.0 * np.pi / box.area * float(up.cpu().item())) + const


def forces_soe(system: ParticleSystem, box: BoxGeometry, params: EwaldParams,
               soe: SOEApprox) -> np.ndarray:
    """Fourier-space forces (nonzero modes + k = 0), input order (369-395)."""
    n = system.n
    if n < 2:
        return np.zeros((n, 3))
    Q = float(np.sum(system.charge ** 2))
    cv, uq = full_sum_constants(params, box, Q)
    bare = BoxGeometry(box.lx, box.ly, box.lz)  # no plane forces in this part
    _, f = device_evaluate(system, bare, params.alpha, params.r_c, soe, params.kmodes, cv, uq,
                           want_forces=True, skip_short_range=True)
    return f


def soe_energy_forces(system: ParticleSystem, box: BoxGeometry, params: EwaldParams,
                      soe: SOEApprox):
    """Full solver evaluation (398-438): (EnergyBreakdown, forces (N,3))."""
    check_short_range_cutoff(box, params.r_c)
    Q = float(np.sum(system.charge ** 2))
    cv, uq = full_sum_constants(params, box, Q)
    e, f = device_evaluate(system, box, params.alpha, params.r_c, soe, params.kmodes, cv, uq)
    return _breakdown(e), f


def total_energy_soe(system: ParticleSystem, box: BoxGeometry, params: EwaldParams,
                     soe: SOEApprox) -> EnergyBreakdown:
    """Energies only (441-452)."""
    check_short_range_cutoff(box, params.r_c)
    Q = float(np.sum(system.charge ** 2))
    cv, uq = full_sum_constants(params, box, Q)
    e, _ = device_evaluate(system, box, params.alpha, params.r_c, soe, params.kmodes, cv, uq,
                           want_forces=False)
    return _breakdown(e)
