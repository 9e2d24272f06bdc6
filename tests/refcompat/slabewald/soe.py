"""``slabewald.soe`` for the reference's tests: this package's SOE module plus
the pointwise closed forms ``xi_soe`` / ``dxi_soe`` (reference soe.py:195-233;
diagnostics outside the hot path) restated in numpy.

For one mode k (> 0) and heights z, with b_l = alpha s_l and
c = 2 alpha / sqrt(pi) e^{-k^2 / (4 alpha^2)}, the exponential sums stand in for
exp(+-kz) erfc(k/2a +- a z):

  xi_+(z) = c Re sum_l w_l e^{-b_l z} / (b_l + k)
  xi_-(z) = c Re sum_l w_l [ e^{-kz} / (b_l + k) + g_l(z) ],
  g_l(z)  = (e^{-kz} - e^{-b_l z}) / (b_l - k) = z e^{-kz} (1 - e^{-u}) / u,
            u = (b_l - k) z,

the last form evaluated by its Taylor series near u = 0 (the removable
singularity at b_l = k).  Derivatives: d/dz of the same sums.
"""

import numpy as np

from paper_2403_01521_b200.soe import *  # noqa: F401,F403
from paper_2403_01521_b200 import soe as _soe

for _k, _v in vars(_soe).items():  # private helpers the tests may reach for
    if _k.startswith("_") and not _k.startswith("__"):
        globals().setdefault(_k, _v)

_SQRT_PI = np.sqrt(np.pi)


def _one_minus_exp_over(u):
    """(1 - e^{-u}) / u for complex u, series below |u| = 1e-2 (error < 1e-17)."""
    u = np.asarray(u, dtype=np.complex128)
    small = np.abs(u) < 1e-2
    safe = np.where(small, 1.0, u)
    direct = (1.0 - np.exp(-safe)) / safe
    series = 1.0 - u / 2.0 + u ** 2 / 6.0 - u ** 3 / 24.0 + u ** 4 / 120.0 - u ** 5 / 720.0
    return np.where(small, series, direct)


def _terms(soe, alpha, k, z):
    if k <= 0:
        raise ValueError("k must be positive (zero mode handled separately)")
    z = np.asarray(z, dtype=np.float64)
    b = alpha * np.asarray(soe.s, dtype=np.complex128)
    w = np.asarray(soe.w, dtype=np.complex128)
    c = 2.0 * alpha / _SQRT_PI * np.exp(-k * k / (4.0 * alpha * alpha))
    zz = z[..., None]
    e_b = np.exp(-b * zz)                     # (..., m)
    e_k = np.exp(-k * z)[..., None]
    g = zz * e_k * _one_minus_exp_over((b - k) * zz)
    return z, b, w, c, e_b, e_k, g


def xi_soe(soe, alpha: float, k: float, z):
    z, b, w, c, e_b, e_k, g = _terms(soe, alpha, k, z)
    xp = c * np.real(np.sum(w / (b + k) * e_b, axis=-1))
    xm = c * np.real(np.sum(w * (e_k / (b + k) + g), axis=-1))
    return xp, xm


def dxi_soe(soe, alpha: float, k: float, z):
    z, b, w, c, e_b, e_k, g = _terms(soe, alpha, k, z)
    # d/dz e^{-bz} = -b e^{-bz};  g' = (b e^{-bz} - k e^{-kz}) / (b - k) = e^{-bz} - k g
    dxp = -c * np.real(np.sum(w * b / (b + k) * e_b, axis=-1))
    dxm = c * np.real(np.sum(w * (-k * e_k / (b + k) - k * g + e_b), axis=-1))
    return dxp, dxm
