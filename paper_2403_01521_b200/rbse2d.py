"""Random-batch SOE Ewald2D (RBSE2D): constants, device mode sampler, estimators.

Drop-in for reference ``pkg/src/slabewald/rbse2d.py``:
  * ``normalization_H`` 46-74, ``charge_term_sum`` 77-89 -- per-run host constants
    (same Poisson-dual / direct branches, same warnings and errors)
  * ``ModeSampler`` 151-207, ``metropolis_batch`` 210-214 -- the Metropolis
    independence chain runs on device (``slab_sample_modes``) with a
    counter-based Philox4x32-10 stream (deterministic per seed; not the numpy
    stream, so draws differ from the reference's while the chain law is the same)
  * ``rb_energy_estimate`` 244-251, ``rb_force_estimate`` 254-271,
    ``rb_energy_forces`` 274-317 -- one ``slab_evaluate`` per call
  * ``run_many_batches`` 332-363, ``variance_diagnostics`` 366-382,
    ``write_diagnostics_csv`` 385-391 -- diagnostics over many batches
"""

from __future__ import annotations

import math
import warnings

import numpy as np
from scipy.special import erfc

from .core import BoxGeometry, EwaldParams, ParticleSystem, enumerate_kmodes
from .soe import SOEApprox
from .ewald2d import raise_on_status
from .soewald2d import _breakdown, device_evaluate

SQRT_PI = math.sqrt(math.pi)
TWO_OVER_SQRT_PI = 2.0 / SQRT_PI


def normalization_H(alpha: float, box: BoxGeometry) -> float:
    """H = sum_{k != 0} exp(-k^2 / 4 alpha^2) via the faster side of Poisson summation."""
    if alpha <= 0:
        raise ValueError("alpha must be positive")
    lmin = min(box.lx, box.ly)
    if alpha * lmin < 5.0:
        warnings.warn("alpha * min(lx, ly) < 5: few Fourier modes carry weight, the "
                      "stochastic mode estimator is inefficient in this regime", stacklevel=2)

    def axis_sum(c, m):
        return float(np.sum(np.exp(-(c * np.arange(-m, m + 1)) ** 2)))

    if alpha * lmin >= 2.0:
        mx = int(np.ceil(7.0 / (alpha * box.lx))) + 1
        my = int(np.ceil(7.0 / (alpha * box.ly))) + 1
        dual = axis_sum(alpha * box.lx, mx) * axis_sum(alpha * box.ly, my)
        return alpha ** 2 * box.area / np.pi * dual - 1.0
    cx, cy = np.pi / (alpha * box.lx), np.pi / (alpha * box.ly)
    mx = int(np.ceil(7.0 / cx)) + 1
    my = int(np.ceil(7.0 / cy)) + 1
    return axis_sum(cx, mx) * axis_sum(cy, my) - 1.0


def charge_term_sum(alpha: float, box: BoxGeometry, Q: float, s_cap: float = 6.0) -> float:
    """C_Q = sum_{0 < |k| <= 2 s_cap alpha} pi Q erfc(k / 2 alpha) / (k A)."""
    km = enumerate_kmodes(box, 2.0 * s_cap * alpha)
    if km.shape[0] == 0:
        return 0.0
    kn = km[:, 2]
    return float(np.sum(np.pi * Q / (kn * box.area) * erfc(kn / (2 * alpha))))


def _axis_logq(m, ax):
    """log proposal mass of the rounded-normal draw on one axis (rbse2d.py:96-102)."""
    am = abs(int(m))
    if am == 0:
        return math.log(math.erf(0.5 * ax))
    # tail-stable erfc difference (the device sampler uses the same form); mass 0 -> -inf
    mass = 0.5 * (math.erfc((am - 0.5) * ax) - math.erfc((am + 0.5) * ax))
    return math.log(mass) if mass > 0 else -math.inf


class ModeSampler:
    """Thinned Metropolis chain over the nonzero integer mode lattice, on device.

    Chain state (mx, my, steps since the last record, RNG counter, accepted,
    steps) lives in a device int64[6]; ``batch`` returns numpy like the
    reference, ``batch_device`` leaves the (P,3) k-set on the device.
    """

    def __init__(self, alpha: float, box: BoxGeometry, seed: int = 0, thin: int = 10,
                 burn_in: int = 100):
        if thin < 1:
            raise ValueError("thin must be at least 1")
        self.alpha = alpha
        self.box = box
        self.thin = int(thin)
        self.seed = int(seed) & 0xFFFFFFFFFFFFFFFF
        self.axx = np.pi / (alpha * box.lx)
        self.axy = np.pi / (alpha * box.ly)
        from .engine import get_engine, require_cuda
        torch = require_cuda()
        self._eng = get_engine()
        self._state = torch.zeros(6, dtype=torch.int64, device=self._eng.device)
        self._eng.sample_modes(self._state, self.seed, alpha, box.lx, box.ly, self.thin,
                               max(int(burn_in), 0), 0)

    @property
    def accepted(self) -> int:
        return int(self._state[4].item())

    @property
    def steps(self) -> int:
        return int(self._state[5].item())

    @property
    def acceptance_rate(self) -> float:
        s = self.steps
        return self.accepted / s if s else float("nan")

    def batch_device(self, P: int, with_indices: bool = False):
        import torch
        modes = torch.empty((P, 3), dtype=torch.float64, device=self._eng.device)
        idx = torch.empty((P, 2), dtype=torch.int64, device=self._eng.device) if with_indices \
            else None
        self._eng.sample_modes(self._state, self.seed, self.alpha, self.box.lx, self.box.ly,
                               self.thin, 0, P, modes, idx)
        return (modes, idx) if with_indices else modes

    def batch_indices(self, P: int) -> np.ndarray:
        """P integer modes (mx, my); repeats carry their multiplicity."""
        _, idx = self.batch_device(int(P), with_indices=True)
        return idx.cpu().numpy()

    def batch(self, P: int) -> np.ndarray:
        """P modes as (kx, ky, |k|) rows (kx = 2 pi mx / lx, |k| = hypot), formed on
        the host from the device-drawn integer indices exactly as rbse2d.py:205-207."""
        rec = self.batch_indices(int(P))
        kx = 2 * np.pi * rec[:, 0] / self.box.lx
        ky = 2 * np.pi * rec[:, 1] / self.box.ly
        return np.column_stack([kx, ky, np.hypot(kx, ky)])


def metropolis_batch(sampler: ModeSampler, P: int) -> np.ndarray:
    if P < 1:
        raise ValueError("batch size must be at least 1")
    return sampler.batch(P)


def _rb_commonv(H: float, P: int, alpha: float) -> float:
    # importance weight exp(+k^2/4a^2) cancels the Gaussian analytically (rbse2d.py:230-232)
    return (H / P) * TWO_OVER_SQRT_PI * alpha


def rb_energy_estimate(system: ParticleSystem, box: BoxGeometry, alpha: float, soe: SOEApprox,
                       modes: np.ndarray, H: float, c_q: float | None = None) -> float:
    """Single-batch estimate of the nonzero-mode Fourier energy (+ C_Q)."""
    if c_q is None:
        c_q = charge_term_sum(alpha, box, float(np.sum(system.charge ** 2)))
    modes = np.asarray(modes, dtype=np.float64).reshape(-1, 3)
    P = modes.shape[0]
    if system.n < 2 or P == 0:
        return 0.0 + c_q
    e, _ = device_evaluate(system, box, alpha, 1.0, soe, modes, _rb_commonv(H, P, alpha), c_q,
                           want_forces=False, skip_short_range=True)
    return float(e[1])


def rb_force_estimate(system: ParticleSystem, box: BoxGeometry, alpha: float, soe: SOEApprox,
                      modes: np.ndarray, H: float) -> np.ndarray:
    """Nonzero-mode forces of one batch + exact k = 0 and plane forces."""
    modes = np.asarray(modes, dtype=np.float64).reshape(-1, 3)
    P = modes.shape[0]
    _, f = device_evaluate(system, box, alpha, 1.0, soe, modes,
                           _rb_commonv(H, max(P, 1), alpha), 0.0, want_forces=True,
                           skip_short_range=True)
    return f


def rb_energy_forces(system: ParticleSystem, box: BoxGeometry, params: EwaldParams,
                     soe: SOEApprox, sampler, P: int, H: float | None = None,
                     c_q: float | None = None):
    """One stochastic evaluation with a fresh batch (rbse2d.py:274-317).

    ``sampler`` is anything with ``batch(P)`` (our device ``ModeSampler``, or a
    stub returning a fixed k-set); a ``ModeSampler`` hands its k-set over on
    device without a host round trip.
    """
    alpha = params.alpha
    if H is None:
        H = normalization_H(alpha, box)
    if c_q is None:
        c_q = charge_term_sum(alpha, box, float(np.sum(system.charge ** 2)))
    # our ModeSampler hands its batch over on device (no host round trip); any
    # other sampler object (a stub with a fixed k-set) through batch(P)
    modes = sampler.batch_device(int(P)) if isinstance(sampler, ModeSampler) else sampler.batch(P)
    e, f = device_evaluate(system, box, alpha, params.r_c, soe, modes, _rb_commonv(H, P, alpha),
                           c_q)
    return _breakdown(e), f


def run_many_batches(system: ParticleSystem, box: BoxGeometry, params: EwaldParams,
                     soe: SOEApprox, n_batches: int, P: int, seed: int = 0, thin: int = 10,
                     burn_in: int = 100) -> np.ndarray:
    """Total-energy estimates over many independent batches of one frozen configuration."""
    alpha = params.alpha
    H = normalization_H(alpha, box)
    Q = float(np.sum(system.charge ** 2))
    c_q = charge_term_sum(alpha, box, Q)
    e0, _ = device_evaluate(system, box, alpha, params.r_c, soe, np.zeros((0, 3)), 0.0, c_q,
                            want_forces=False)
    u_det = float(e0[0] + e0[2] - e0[3] + e0[4] + c_q)  # u_s + u_l_0 - u_self + u_ps + C_Q
    sampler = ModeSampler(alpha, box, seed=seed, thin=thin, burn_in=burn_in)
    out = np.empty(n_batches)
    if system.n < 2:
        out[:] = 0.0
        return out + u_det
    from .engine import get_engine, to_device
    eng = get_engine()
    pos, q = to_device(system.pos), to_device(system.charge)
    # rbse2d.py:346-363: all n_batches * P modes drawn as one chain continuation,
    # then one batched forward-sweep energy launch sequence (sort and decay
    # table once; ~4096 modes per device pass)
    modes = sampler.batch_device(n_batches * P)
    e, status = eng.batch_energies(pos, q, soe, alpha, box.area, modes, n_batches, P,
                                   _rb_commonv(H, P, alpha))
    raise_on_status(int(status.cpu().item()))
    return e.cpu().numpy() + u_det


def variance_diagnostics(estimates: np.ndarray) -> dict:
    """Mean, standard error and their running versions over a batch series."""
    est = np.asarray(estimates, dtype=np.float64)
    nb = len(est)
    if nb < 2:
        raise ValueError("need at least two batches")
    k = np.arange(1, nb + 1)
    mean_run = np.cumsum(est) / k
    var = np.maximum(np.cumsum(est ** 2) - k * mean_run ** 2, 0.0)
    se_run = np.zeros(nb)
    se_run[1:] = np.sqrt(var[1:] / (k[1:] - 1.0)) / np.sqrt(k[1:])
    return {"n": nb, "mean": float(mean_run[-1]), "stderr": float(se_run[-1]),
            "running_mean": mean_run, "running_stderr": se_run}


def write_diagnostics_csv(path, estimates: np.ndarray) -> None:
    d = variance_diagnostics(estimates)
    lines = ["batch_index,estimate,running_mean,running_stderr"]
    lines += [f"{i},{e:.17g},{m:.17g},{s:.17g}" for i, (e, m, s) in
              enumerate(zip(estimates, d["running_mean"], d["running_stderr"]))]
    with open(path, "w") as fh:
        fh.write("\n".join(lines) + "\n")
