"""ctypes binding of the in-tree C-ABI library ``_lib/libslabewald_b200.so``.

The library is the product: every device computation of this package goes
through it.  There is no CPU fallback -- if the library is missing, or no CUDA
device is visible, every entry point raises ``NativeUnavailable``.
Signatures mirror ``include/slabewald_b200.h``.
"""

from __future__ import annotations

import ctypes
import os

HERE = os.path.dirname(os.path.abspath(__file__))
# SLAB_B200_LIB: alternative build of the same library (kernel-variant A/B timing)
LIB_PATH = os.environ.get("SLAB_B200_LIB") or os.path.join(HERE, "_lib", "libslabewald_b200.so")

SLAB_OK = 0
SLAB_ERR_ARG = 1
SLAB_ERR_CUDA = 2
SLAB_ERR_UNSUPPORTED = 3
SLAB_ERR_NOMEM = 4
SLAB_STATUS_COINCIDENT = 1
SLAB_STATUS_SINGULAR = 2
SLAB_STATUS_NBR_OVERFLOW = 4
SLAB_STATUS_NONFINITE = 8
SLAB_STATUS_WALL = 16
SLAB_SHARD_MODES = 0
SLAB_SHARD_ZSPLIT = 1

EXPORTED = (
    "slab_ctx_create", "slab_ctx_destroy", "slab_last_error", "slab_version",
    "slab_sort_by_z", "slab_fourier_sweep", "slab_zero_mode_sweep", "slab_short_range",
    "slab_sample_modes", "slab_evaluate", "slab_recursive_pair_sum", "slab_fp64_peak",
    "slab_ctx_neighbor_capacity", "slab_ctx_last_max_neighbors", "slab_batch_energies",
    "slab_wca", "slab_walls", "slab_md_langevin", "slab_md_kick", "slab_md_drift",
    "slab_md_scale", "slab_md_kinetic", "slab_zsplit_exchange_doubles",
    "slab_ewald_ref_fourier", "slab_ewald_ref_zero", "slab_evaluate_host", "slab_constant_terms",
)


class NativeUnavailable(RuntimeError):
    """The CUDA library (or a CUDA device) is not available: no fallback exists."""


class SlabBox(ctypes.Structure):
    _fields_ = [("lx", ctypes.c_double), ("ly", ctypes.c_double), ("lz", ctypes.c_double),
                ("sigma_top", ctypes.c_double), ("sigma_bot", ctypes.c_double)]


_DP = ctypes.POINTER(ctypes.c_double)


class SlabSOE(ctypes.Structure):
    _fields_ = [("m", ctypes.c_int), ("h_w_re", _DP), ("h_w_im", _DP), ("h_s_re", _DP),
                ("h_s_im", _DP)]


class SlabEvalArgs(ctypes.Structure):
    _fields_ = [
        ("n", ctypes.c_int64),
        ("d_pos", ctypes.c_void_p),
        ("d_charge", ctypes.c_void_p),
        ("box", SlabBox),
        ("alpha", ctypes.c_double),
        ("r_c", ctypes.c_double),
        ("soe", SlabSOE),
        ("d_modes", ctypes.c_void_p),
        ("nmode", ctypes.c_int64),
        ("d_commonv", ctypes.c_void_p),
        ("commonv_scalar", ctypes.c_double),
        ("charge_const", ctypes.c_double),
        ("want_forces", ctypes.c_int),
        ("skip_short_range", ctypes.c_int),
        ("d_forces", ctypes.c_void_p),
        ("d_energy", ctypes.c_void_p),
        ("d_perm", ctypes.c_void_p),
        ("shard_rank", ctypes.c_int),
        ("shard_count", ctypes.c_int),
        ("ev_scan_begin", ctypes.c_void_p),
        ("ev_scan_end", ctypes.c_void_p),
        ("shard_mode", ctypes.c_int),
        ("phase", ctypes.c_int),
        ("d_xchg", ctypes.c_void_p),
        ("ev_modes_ready", ctypes.c_void_p),
    ]


_lib = None


def load():
    """Load (once) and return the ctypes library; raises NativeUnavailable."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        raise NativeUnavailable(
            f"CUDA library not built: {LIB_PATH} is missing (run __graft_entry__.build() "
            "or `make -C paper_2403_01521_b200/csrc`)")
    lib = ctypes.CDLL(LIB_PATH)
    vp, i64, dbl, cint = ctypes.c_void_p, ctypes.c_int64, ctypes.c_double, ctypes.c_int
    lib.slab_ctx_create.argtypes = [ctypes.POINTER(vp)]
    lib.slab_ctx_destroy.argtypes = [vp]
    lib.slab_last_error.restype = ctypes.c_char_p
    lib.slab_version.restype = ctypes.c_char_p
    lib.slab_sort_by_z.argtypes = [vp, vp, i64, i64, vp, vp]
    lib.slab_fourier_sweep.argtypes = [vp, vp, vp, vp, vp, i64, vp, vp, dbl, i64, SlabSOE, dbl,
                                       dbl, cint, vp, vp, vp, vp]
    lib.slab_zero_mode_sweep.argtypes = [vp, vp, vp, i64, SlabSOE, dbl, cint, vp, vp, vp]
    lib.slab_short_range.argtypes = [vp, vp, vp, i64, SlabBox, dbl, dbl, vp, vp, vp, vp]
    lib.slab_sample_modes.argtypes = [vp, vp, ctypes.c_uint64, dbl, dbl, dbl, cint, cint, i64, vp,
                                      vp, vp]
    lib.slab_evaluate.argtypes = [vp, ctypes.POINTER(SlabEvalArgs), vp]
    lib.slab_evaluate_host.argtypes = [vp, ctypes.POINTER(SlabEvalArgs), vp, vp, vp, vp, vp]
    lib.slab_recursive_pair_sum.argtypes = [vp, vp, vp, vp, i64, dbl, dbl, vp, vp]
    lib.slab_batch_energies.argtypes = [vp, vp, vp, i64, SlabSOE, dbl, dbl, vp, i64, i64, dbl, vp,
                                        vp, vp]
    lib.slab_wca.argtypes = [vp, vp, i64, SlabBox, dbl, dbl, vp, vp, vp, vp]
    lib.slab_walls.argtypes = [vp, vp, i64, dbl, dbl, dbl, vp, vp, vp, vp]
    lib.slab_md_langevin.argtypes = [vp, vp, vp, vp, i64, dbl, dbl, dbl, ctypes.c_uint64, vp, vp,
                                     dbl, dbl, vp]
    lib.slab_md_kick.argtypes = [vp, vp, vp, i64, dbl, vp]
    lib.slab_md_drift.argtypes = [vp, vp, i64, dbl, vp, dbl, dbl, vp]
    lib.slab_md_scale.argtypes = [vp, i64, dbl, vp]
    lib.slab_md_kinetic.argtypes = [vp, vp, vp, i64, vp, vp]
    lib.slab_zsplit_exchange_doubles.argtypes = [i64, cint, cint]
    lib.slab_ewald_ref_fourier.argtypes = [vp, vp, vp, i64, dbl, dbl, dbl, vp, vp, cint, vp, cint,
                                           cint, cint, cint, vp, vp, vp]
    lib.slab_ewald_ref_zero.argtypes = [vp, vp, vp, i64, dbl, vp, vp, vp]
    lib.slab_fp64_peak.argtypes = [ctypes.POINTER(dbl)]
    lib.slab_constant_terms.argtypes = [vp, vp, vp, i64, SlabBox, dbl, vp, vp]
    lib.slab_ctx_neighbor_capacity.argtypes = [vp, cint]
    lib.slab_ctx_last_max_neighbors.argtypes = [vp, ctypes.POINTER(cint)]

    for name in EXPORTED:
        if name not in ("slab_last_error", "slab_version", "slab_zsplit_exchange_doubles"):
            getattr(lib, name).restype = cint
    lib.slab_zsplit_exchange_doubles.restype = i64
    _lib = lib
    return lib


def check(rc: int, what: str):
    if rc != SLAB_OK:
        msg = load().slab_last_error().decode()
        if rc == SLAB_ERR_UNSUPPORTED:
            raise NotImplementedError(f"{what}: {msg}")
        if rc == SLAB_ERR_ARG:
            raise ValueError(f"{what}: {msg}")
        raise RuntimeError(f"{what} failed ({rc}): {msg}")
