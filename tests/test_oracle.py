"""CPU: the C oracle (oracle/slab_oracle.c) pinned against the REAL reference.

tests/golden/*.npz were produced by running the reference package on these same
seeded inputs (tests/golden/make_golden.py).  The oracle must reproduce them
essentially bit-for-bit (it restates the numba loops in the same order): we
require 1e-13 relative on energies and 1e-13 of max|F| on forces -- three
orders tighter than the GPU bar -- and exact permutations.
"""

import hashlib

import numpy as np
import pytest

from helpers import load_golden
from oracle import oracle as O
from paper_2403_01521_b200.configs import make_workload


def _sha(a):
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


@pytest.mark.parametrize("name", ["small_600", "small_2000", "cfg1", "cfg2", "cfg5_1e4"])
def test_oracle_matches_reference_goldens(name):
    g = load_golden(name)
    wl = make_workload(name)
    assert _sha(wl.system.pos) == str(g["pos_sha"])
    P = int(g["P"])
    modes = g["modes"]
    if P == 0:
        cv = O.full_commonv(modes[:, 2], wl.alpha)
        cc = O.full_uq(modes[:, 2], float(np.sum(wl.system.charge ** 2)), wl.box.area, wl.alpha)
    else:
        cv = O.rb_commonv(float(g["H"]), P, wl.alpha)
        cc = float(g["c_q"])
    e, f, flag = O.energy_forces(wl.system.pos, wl.system.charge, wl.box, wl.alpha,
                                 wl.params().r_c, modes, cv, cc, g["soe_w"], g["soe_s"])
    assert flag == 0
    for val, key in zip(e, ("u_s", "u_l_k", "u_l_0", "u_self", "u_ps")):
        ref = float(g[key])
        assert abs(val - ref) <= 1e-13 * max(abs(ref), 1.0), (key, val, ref)
    fmax = float(g["fmax"])
    assert np.max(np.abs(f - g["forces"])) <= 1e-13 * fmax


@pytest.mark.parametrize("name", ["small_600", "cfg1", "cfg2"])
def test_oracle_short_range_matches_reference(name):
    g = load_golden(name)
    wl = make_workload(name)
    u, f, flag = O.short_range(wl.system.pos, wl.system.charge, wl.box, wl.alpha,
                               wl.params().r_c)
    assert flag == 0
    assert abs(u - float(g["u_s_alone"])) <= 1e-13 * abs(float(g["u_s_alone"]))
    assert np.max(np.abs(f - g["f_short"])) <= 1e-13 * np.max(np.abs(g["f_short"]))


def test_oracle_sort_matches_reference_cases():
    g = load_golden("units")
    cases = sorted({k[:-2] for k in g if k.startswith("sort_") and k.endswith("_z")})
    assert len(cases) >= 6
    for c in cases:
        z, lz, want = g[c + "_z"], float(g[c + "_lz"]), g[c + "_perm"]
        got = O.sort_perm(z, lz)
        np.testing.assert_array_equal(got, want, err_msg=c)
        np.testing.assert_array_equal(got, np.argsort(z, kind="stable"), err_msg=c)


def test_oracle_sort_known_answers():
    # reference tests/test_core.py:196-217
    np.testing.assert_array_equal(O.sort_perm([3.0, 1.0, 2.0], 4.0), [1, 2, 0])
    np.testing.assert_array_equal(O.sort_perm([1.0, 0.25, 1.0, 0.25, 1.0], 2.0),
                                  [1, 3, 0, 2, 4])
    np.testing.assert_array_equal(O.sort_perm([0.5, 1.0, 2.0, 3.5], 4.0), [0, 1, 2, 3])


def test_oracle_large_config_perm_hashes():
    for name in ("cfg3", "cfg5_1e5"):
        g = load_golden(name)
        wl = make_workload(name)
        perm = O.sort_perm(wl.system.pos[:, 2], wl.box.lz)
        assert _sha(perm) == str(g["perm_sha"]), name


def test_oracle_batch_energies_match_reference():
    """The oracle's forward sweep (energy only) per injected batch equals the
    reference's _rb_batch_energy_kernel (tests/golden/batches.npz)."""
    from oracle import oracle as O
    from paper_2403_01521_b200.configs import make_workload
    from paper_2403_01521_b200.soe import build_soe_contour
    g = load_golden("batches")
    wl = make_workload("cfg5_1e4")
    soe = build_soe_contour(wl.m)
    perm = O.sort_perm(wl.system.pos[:, 2], wl.box.lz)
    xs, ys, zs = (np.ascontiguousarray(wl.system.pos[perm, i]) for i in range(3))
    qs = wl.system.charge[perm]
    P = int(g["P"])
    cv = O.rb_commonv(float(g["H"]), P, wl.alpha)
    scale = np.max(np.abs(g["batch_u"]))
    for b in (0, 17, int(g["n_batches"]) - 1):
        u, _ = O.fourier_sweep(xs, ys, zs, qs, g["modes"][b * P:(b + 1) * P], cv, soe.w, soe.s,
                               wl.alpha, wl.box.area, nthreads=4)
        assert abs(u - g["batch_u"][b]) <= 1e-12 * scale, b


def test_oracle_lone_complex_soe_table_matches_reference():
    """A table with lone complex terms (no conjugate partners) through the oracle's
    full mode sum equals the reference's soe_energy_forces (golden lone_soe)."""
    from paper_2403_01521_b200.core import BoxGeometry, make_ewald_params, make_system
    from paper_2403_01521_b200.soewald2d import full_sum_constants
    g = load_golden("lone_soe")
    box = BoxGeometry(*[float(v) for v in g["box"]])
    s = make_system(g["q"], np.ones(len(g["q"])), g["pos"], box=box)
    params = make_ewald_params(float(g["alpha"]), float(g["s_par"]), box)
    cv, uq = full_sum_constants(params, box, float(np.sum(s.charge ** 2)))
    e, f, flag = O.energy_forces(s.pos, s.charge, box, params.alpha, params.r_c, params.kmodes,
                                 cv, uq, g["w"], g["s"])
    for val, key in zip(e, ("u_s", "u_l_k", "u_l_0", "u_self", "u_ps")):
        assert val == pytest.approx(float(g[key]), rel=1e-13, abs=1e-13), key
    assert np.max(np.abs(f - g["forces"])) <= 1e-13 * np.max(np.abs(g["forces"]))
