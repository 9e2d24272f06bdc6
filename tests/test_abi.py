"""CPU: the C-ABI library loads and exports every entry point include/*.h declares,
and the product path refuses to run without a GPU (no CPU fallback)."""

import ctypes
import os
import re

import pytest

from paper_2403_01521_b200 import _native

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _declared():
    src = open(os.path.join(REPO, "include", "slabewald_b200.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(?:int|int64_t|const char\*)\s+(slab_\w+)\s*\(", src)))


def test_header_declares_the_boundary():
    names = _declared()
    for must in ("slab_evaluate", "slab_sort_by_z", "slab_fourier_sweep", "slab_zero_mode_sweep",
                 "slab_short_range", "slab_sample_modes", "slab_recursive_pair_sum"):
        assert must in names


def test_library_exports_every_declared_symbol():
    if not os.path.exists(_native.LIB_PATH):
        pytest.skip("library not built (run __graft_entry__.build())")
    lib = ctypes.CDLL(_native.LIB_PATH)
    for name in _declared():
        assert hasattr(lib, name), name
    assert set(_declared()) == set(_native.EXPORTED)
    v = _native.load().slab_version().decode()
    assert "sm_100a" in v


def test_eval_struct_matches_header_field_order():
    src = open(os.path.join(REPO, "include", "slabewald_b200.h")).read()
    body = src[src.index("typedef struct SlabEvalArgs"):src.index("} SlabEvalArgs;")]
    body = re.sub(r"/\*.*?\*/", "", body, flags=re.S)
    fields = re.findall(r"\b(\w+)\s*;", body)
    assert fields == [f[0] for f in _native.SlabEvalArgs._fields_]


def test_no_cpu_fallback_without_gpu():
    import torch
    if torch.cuda.is_available():
        pytest.skip("a GPU is present")
    import numpy as np
    import paper_2403_01521_b200 as pk
    box = pk.BoxGeometry(20.0, 20.0, 10.0)
    s = pk.make_system([1.0, -1.0], [1.0, 1.0], [[1, 1, 1], [5, 5, 5]], box)
    params = pk.make_ewald_params(0.5, 3.0, box)
    soe = pk.build_soe_contour(8)
    with pytest.raises(_native.NativeUnavailable):
        pk.soe_energy_forces(s, box, params, soe)
    with pytest.raises(_native.NativeUnavailable):
        pk.sort_by_z(s, box.lz)
