"""ctypes front-end of the C oracle (``oracle/slab_oracle.c``).

TEST INFRASTRUCTURE ONLY -- imported by tests/, ``__graft_entry__.smoke()`` and
bench.py's CPU-baseline legs, never by the product package.  Each wrapper
takes the same numpy arrays as the reference function it restates.
"""

from __future__ import annotations

import ctypes
import os
import subprocess

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "liboracle.so")
_lib = None

_D = ctypes.POINTER(ctypes.c_double)
_I64 = ctypes.POINTER(ctypes.c_int64)


def build():
    subprocess.run(["make", "-s", "-C", HERE], check=True)


def lib():
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            build()
        L = ctypes.CDLL(LIB_PATH)
        i64, dbl, cint = ctypes.c_int64, ctypes.c_double, ctypes.c_int
        L.oracle_sort_perm.argtypes = [_D, i64, dbl, _I64]
        L.oracle_sort_perm.restype = None
        L.oracle_short_range.argtypes = [_D, _D, i64, dbl, dbl, dbl, dbl, dbl, _D,
                                         ctypes.POINTER(cint), cint]
        L.oracle_short_range.restype = dbl
        L.oracle_energy_forces.argtypes = ([_D, _D, i64] + [dbl] * 7 + [_D, _D, _D, _D, i64, dbl]
                                           + [_D] * 4 + [cint, cint, _D, _D])
        L.oracle_energy_forces.restype = cint
        L.oracle_decay_table.argtypes = [_D, i64, _D, _D, cint, _D, _D]
        L.oracle_decay_table.restype = None
        L.oracle_fourier_sweep_mt.argtypes = ([_D] * 4 + [i64] + [_D] * 4 + [i64] + [_D] * 4
                                              + [cint, dbl, _D, _D, cint, _D, cint])
        L.oracle_fourier_sweep_mt.restype = dbl
        L.oracle_zero_mode_sweep.argtypes = ([_D, _D, i64] + [_D] * 6 + [cint, dbl, dbl, _D, _D,
                                                                       cint, _D])
        L.oracle_zero_mode_sweep.restype = dbl
        L.oracle_short_range_home.argtypes = [_D, _D, i64, dbl, dbl, dbl, dbl, dbl, i64, i64, _D,
                                              ctypes.POINTER(cint)]
        L.oracle_short_range_home.restype = dbl
        _lib = L
    return _lib


def _p(a):
    return a.ctypes.data_as(_D)


def _c(a, dt=np.float64):
    return np.ascontiguousarray(a, dtype=dt)


def sort_perm(z, lz) -> np.ndarray:
    """core.py:166-200 bucket sort (stable ascending z)."""
    z = _c(z)
    perm = np.empty(len(z), dtype=np.int64)
    lib().oracle_sort_perm(_p(z), len(z), float(lz), perm.ctypes.data_as(_I64))
    return perm


def short_range(pos, charge, box, alpha, r_c, nthreads=1):
    """ewald2d.py:280-303 (u_s, forces, flag); no ValueError mapping here."""
    pos, charge = _c(pos), _c(charge)
    f = np.zeros((len(charge), 3))
    flag = ctypes.c_int(0)
    u = lib().oracle_short_range(_p(pos), _p(charge), len(charge), box.lx, box.ly, box.lz,
                                 float(alpha), float(r_c), _p(f), ctypes.byref(flag),
                                 int(nthreads))
    return u, f, flag.value


def short_range_home(pos, charge, box, alpha, r_c, h0, h1):
    """Shard share of the short range (tests of the multi-GPU decomposition)."""
    pos, charge = _c(pos), _c(charge)
    f = np.zeros((len(charge), 3))
    flag = ctypes.c_int(0)
    u = lib().oracle_short_range_home(_p(pos), _p(charge), len(charge), box.lx, box.ly, box.lz,
                                      float(alpha), float(r_c), int(h0), int(h1), _p(f),
                                      ctypes.byref(flag))
    return u, f, flag.value


def fourier_sweep(x, y, z, q, modes, commonv, soe_w, soe_s, alpha, area, nthreads=1):
    """soewald2d.py:85-208 on sorted arrays: (energy, forces_sorted)."""
    x, y, z, q = (_c(a) for a in (x, y, z, q))
    modes = _c(modes).reshape(-1, 3)
    kx, ky, kv = (_c(modes[:, i]) for i in range(3))
    commonv = _c(commonv)
    w = np.asarray(soe_w, dtype=np.complex128)
    b = alpha * np.asarray(soe_s, dtype=np.complex128)
    wr, wi, br, bi = _c(w.real), _c(w.imag), _c(b.real), _c(b.imag)
    n, m = len(q), len(w)
    dr, di = np.zeros(n * m), np.zeros(n * m)
    lib().oracle_decay_table(_p(z), n, _p(br), _p(bi), m, _p(dr), _p(di))
    f = np.zeros((n, 3))
    u = lib().oracle_fourier_sweep_mt(_p(x), _p(y), _p(z), _p(q), n, _p(kx), _p(ky), _p(kv),
                                      _p(commonv), len(kv), _p(wr), _p(wi), _p(br), _p(bi), m,
                                      float(area), _p(dr), _p(di), 1, _p(f), int(nthreads))
    return u, f


def energy_forces(pos, charge, box, alpha, r_c, modes, commonv, charge_const, soe_w, soe_s,
                  nthreads=1):
    """Assembly of rbse2d.py:274-317 / soewald2d.py:398-438 for an explicit k-set.

    Returns ([u_s, u_l_k, u_l_0, u_self, u_ps], forces (N,3), flag)."""
    pos, charge = _c(pos), _c(charge)
    modes = _c(modes).reshape(-1, 3)
    kx, ky, kv = (_c(modes[:, i]) for i in range(3))
    commonv = _c(commonv)
    w = np.asarray(soe_w, dtype=np.complex128)
    s = np.asarray(soe_s, dtype=np.complex128)
    wr, wi, sr, si = _c(w.real), _c(w.imag), _c(s.real), _c(s.imag)
    n = len(charge)
    e = np.zeros(5)
    f = np.zeros((n, 3))
    flag = lib().oracle_energy_forces(
        _p(pos), _p(charge), n, box.lx, box.ly, box.lz, box.sigma_top, box.sigma_bot,
        float(alpha), float(r_c), _p(kx), _p(ky), _p(kv), _p(commonv), len(kv),
        float(charge_const), _p(wr), _p(wi), _p(sr), _p(si), len(w), int(nthreads), _p(e), _p(f))
    return e, f, flag


def rb_commonv(H, P, alpha):
    """rbse2d.py:301: (H/P)(2 alpha/sqrt(pi)) for every sampled mode."""
    return np.full(P, (H / P) * (2.0 / np.sqrt(np.pi)) * alpha)


def full_commonv(knorm, alpha):
    """soewald2d.py:421-422: (2 alpha/sqrt(pi)) exp(-k^2/4 alpha^2)."""
    return (2.0 / np.sqrt(np.pi)) * alpha * np.exp(-np.asarray(knorm) ** 2 / (4 * alpha ** 2))


def full_uq(knorm, Q, area, alpha):
    """soewald2d.py:408-413 deterministic charge term of the full mode sum."""
    from scipy.special import erfc
    knorm = np.asarray(knorm)
    return float(np.sum(np.pi * Q / (knorm * area) * erfc(knorm / (2 * alpha))))
