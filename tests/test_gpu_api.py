"""GPU: the drop-in API through the CUDA library, mirroring the reference's own
test strategy (pkg/tests/test_soewald2d.py, test_rbse2d.py, test_core.py,
test_ewald2d.py): known answers, O(N^2) relational checks, finite-difference
gradients, statistics of the sampler, error messages.  Every call below runs
the sm_100a kernels (there is no CPU path)."""

import math

import numpy as np
import pytest
from scipy.special import erfc
from scipy.stats import chisquare

from helpers import StubSampler, load_golden

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def pk():
    import paper_2403_01521_b200 as pk
    return pk


def _slab_system(pk, n_pairs, box, seed, margin=0.5):
    rng = np.random.default_rng(seed)
    n = 2 * n_pairs
    pos = rng.uniform([0.0, 0.0, margin], [box.lx, box.ly, box.lz - margin], size=(n, 3))
    charge = np.array([1.0, -1.0] * n_pairs)
    return pk.make_system(charge, np.ones(n), pos, box)


def _numerical_gradient(f, pos, h=1e-5):
    pos = np.array(pos, dtype=np.float64)
    grad = np.zeros_like(pos)
    for i in range(pos.shape[0]):
        for d in range(3):
            keep = pos[i, d]
            pos[i, d] = keep + h
            up = f(pos)
            pos[i, d] = keep - h
            dn = f(pos)
            pos[i, d] = keep
            grad[i, d] = (up - dn) / (2 * h)
    return grad


# --------------------------------------------------------------- recursion
def test_recursion_known_answers(pk):
    out = pk.recursive_pair_sum(np.array([2.0]), np.array([0.3]), np.array([1.0]), 0.5 + 0j)
    assert out.shape == (1,) and out[0] == 0.0
    q = np.array([1.0, 1.0])
    th = np.array([0.7, 0.7])
    a = pk.recursive_pair_sum(q, th, np.array([0.0, 1.0]), complex(np.log(2.0)))
    s = np.sum(q * np.exp(1j * th) * a)
    assert s.real == pytest.approx(0.5, rel=1e-14) and abs(s.imag) <= 1e-15


def test_recursion_matches_reference_golden_and_direct(pk):
    g = load_golden("units")
    q, th, z = g["rps_q"], g["rps_theta"], g["rps_z"]
    for j in range(3):
        beta = complex(g[f"rps_{j}_beta"])
        got = pk.recursive_pair_sum(q, th, z, beta)
        want = g[f"rps_{j}_out"]
        scale = max(1.0, float(np.max(np.abs(want))))
        np.testing.assert_allclose(got, want, rtol=0, atol=1e-12 * scale)
        # O(N^2) direct evaluation (reference tests/oracles.py:127-143)
        direct = np.array([np.sum(q[:a] * np.exp(-1j * th[:a] - beta * (z[a] - z[:a])))
                           for a in range(len(z))])
        np.testing.assert_allclose(got, direct, rtol=0, atol=1e-12 * scale)


def test_recursion_errors(pk):
    with pytest.raises(ValueError, match="sorted"):
        pk.recursive_pair_sum(np.ones(3), np.zeros(3), np.array([0.0, 2.0, 1.0]), 1.0 + 0j)
    with pytest.raises(ValueError, match="nonnegative"):
        pk.recursive_pair_sum(np.ones(2), np.zeros(2), np.array([0.0, 1.0]), -0.1 + 1.0j)


# --------------------------------------------------------------- sort
def test_sort_cases_bit_exact(pk):
    g = load_golden("units")
    cases = sorted({k[:-2] for k in g if k.startswith("sort_") and k.endswith("_z")})
    for c in cases:
        z, lz, want = g[c + "_z"], float(g[c + "_lz"]), g[c + "_perm"]
        pos = np.column_stack([np.zeros(len(z)), np.zeros(len(z)), z])
        s = pk.make_system(np.ones(len(z)), np.ones(len(z)), pos)
        np.testing.assert_array_equal(pk.sort_by_z(s, lz), want, err_msg=c)


def test_sort_negative_and_nonfinite(pk):
    z = np.array([0.5, -1.0, 0.0, -0.0, -1.0, 2.0])
    pos = np.column_stack([np.zeros(6), np.zeros(6), z])
    s = pk.make_system(np.ones(6), np.ones(6), pos)
    np.testing.assert_array_equal(pk.sort_by_z(s, 3.0), np.argsort(z, kind="stable"))
    pos[1, 2] = np.nan
    with pytest.raises(ValueError, match="finite"):
        pk.sort_by_z(pk.make_system(np.ones(6), np.ones(6), pos), 3.0)


def test_sort_large_random_bijection(pk):
    z = np.random.default_rng(4).random(300_001) * 6.0
    pos = np.column_stack([np.zeros_like(z), np.zeros_like(z), z])
    s = pk.make_system(np.ones(len(z)), np.ones(len(z)), pos)
    np.testing.assert_array_equal(pk.sort_by_z(s, 6.0), np.argsort(z, kind="stable"))


# --------------------------------------------------------------- per-mode / zero mode
def test_mode_energies_and_zero_mode_match_reference(pk):
    g = load_golden("units")
    box = pk.BoxGeometry(20.0, 20.0, 10.0)
    s = pk.make_system(g["mode_q"], np.ones(20), g["mode_pos"], box)
    params = pk.make_ewald_params(0.5, 3.0, box)
    soe8 = pk.build_soe_contour(8)
    got = np.array([pk.fourier_mode_energy_soe(s, box, params, soe8, i)
                    for i in range(params.kmodes.shape[0])])
    ref = g["mode_energies"]
    np.testing.assert_allclose(got, ref, rtol=1e-10, atol=1e-12 * np.max(np.abs(ref)))
    z0 = pk.zero_mode_energy_soe(s, box, 0.5, soe8)
    assert z0 == pytest.approx(float(g["mode_zero"]), rel=1e-10)
    bd, f = pk.soe_energy_forces(s, box, params, soe8)
    assert bd.total == pytest.approx(float(g["mode_total"]), rel=1e-10)
    np.testing.assert_allclose(f, g["mode_forces"], rtol=0,
                               atol=1e-9 * np.max(np.abs(g["mode_forces"])))
    np.testing.assert_allclose(pk.forces_soe(s, box, params, soe8), g["mode_forces_soe"], rtol=0,
                               atol=1e-9 * np.max(np.abs(g["mode_forces_soe"])))


def test_single_particle_mode_energy_is_charge_term(pk):
    box = pk.BoxGeometry(20.0, 20.0, 10.0)
    s = pk.make_system([1.0], [1.0], [[3.0, 4.0, 5.0]], box)
    params = pk.make_ewald_params(0.5, 3.0, box)
    soe8 = pk.build_soe_contour(8)
    for idx in (0, 3):
        k = params.kmodes[idx, 2]
        want = np.pi * erfc(k / 1.0) / (k * box.area)
        assert pk.fourier_mode_energy_soe(s, box, params, soe8, idx) == pytest.approx(want,
                                                                                   rel=1e-13)
    with pytest.raises(IndexError, match="mode index"):
        pk.fourier_mode_energy_soe(s, box, params, soe8, params.kmodes.shape[0])


def test_zero_mode_equal_heights(pk):
    box = pk.BoxGeometry(12.0, 9.0, 6.0)
    charge = np.array([1.0, -2.0, 1.0])
    pos = np.array([[1.0, 1.0, 2.5], [4.0, 7.0, 2.5], [9.0, 3.0, 2.5]])
    s = pk.make_system(charge, np.ones(3), pos, box)
    soe8 = pk.build_soe_contour(8)
    alpha = 0.7
    g0 = complex(np.sum(soe8.w)).real / (alpha * math.sqrt(math.pi))
    want = (-2.0 * np.pi / box.area) * -3.0 * g0 - math.sqrt(math.pi) * 6.0 / (alpha * box.area)
    assert pk.zero_mode_energy_soe(s, box, alpha, soe8) == pytest.approx(want, rel=1e-13)


def test_presorted_paths_match_full(pk):
    box = pk.BoxGeometry(20.0, 20.0, 10.0)
    s = _slab_system(pk, 15, box, 5)
    params = pk.make_ewald_params(0.5, 3.0, box)
    soe = pk.build_soe_contour(16)
    perm = np.argsort(s.pos[:, 2], kind="stable")
    pre = (s.pos[perm, 0], s.pos[perm, 1], s.pos[perm, 2], s.charge[perm])
    a = pk.fourier_energy_soe(s, box, params, soe)
    b = pk.fourier_energy_soe(s, box, params, soe, _presorted=pre)
    assert a == pytest.approx(b, rel=1e-12)
    za = pk.zero_mode_energy_soe(s, box, 0.5, soe)
    zb = pk.zero_mode_energy_soe(s, box, 0.5, soe, _presorted=pre)
    assert za == pytest.approx(zb, rel=1e-12)
    bad = (pre[0], pre[1], pre[2][::-1].copy(), pre[3])
    with pytest.raises(ValueError, match="sorted ascending"):
        pk.fourier_energy_soe(s, box, params, soe, _presorted=bad)


# --------------------------------------------------------------- forces
def test_forces_are_exact_gradient(pk):
    box = pk.BoxGeometry(10.0, 10.0, 6.0)
    s = _slab_system(pk, 8, box, 41, margin=0.8)
    params = pk.make_ewald_params(0.8, 3.0, box)
    soe8 = pk.build_soe_contour(8)
    _, forces = pk.soe_energy_forces(s, box, params, soe8)

    def energy(pos):
        moved = pk.make_system(s.charge, s.mass, pos, box)
        return pk.total_energy_soe(moved, box, params, soe8).total

    grad = _numerical_gradient(energy, s.pos)
    np.testing.assert_allclose(forces, -grad, rtol=0, atol=1e-5 * np.max(np.abs(forces)))


def test_two_particle_forces_antisymmetric(pk):
    box = pk.BoxGeometry(10.0, 10.0, 6.0)
    s = pk.make_system([1.0, -1.0], np.ones(2), [[1.2, 3.4, 1.7], [6.8, 5.1, 4.2]], box)
    f = pk.forces_soe(s, box, pk.make_ewald_params(0.8, 3.0, box), pk.build_soe_contour(8))
    np.testing.assert_allclose(f[0], -f[1], rtol=0, atol=5e-14 * np.max(np.abs(f)))


def test_rb_force_estimate_is_gradient_of_frozen_batch(pk):
    box = pk.BoxGeometry(10.0, 10.0, 5.0, sigma_top=0.003, sigma_bot=-0.001)
    s = _slab_system(pk, 5, box, 63, margin=0.8)
    alpha = 0.8
    soe8 = pk.build_soe_contour(8)
    import warnings
    with warnings.catch_warnings():
        warnings.simplefilter("ignore")
        H = pk.normalization_H(alpha, box)
    modes = pk.ModeSampler(alpha, box, seed=9).batch(8)
    forces = pk.rb_force_estimate(s, box, alpha, soe8, modes, H)

    def energy(pos):
        m = pk.make_system(s.charge, s.mass, pos, box)
        return (pk.rb_energy_estimate(m, box, alpha, soe8, modes, H, c_q=0.0)
                + pk.zero_mode_energy_soe(m, box, alpha, soe8) + pk.slab_energy_forces(m, box)[0])

    grad = _numerical_gradient(energy, s.pos)
    np.testing.assert_allclose(forces, -grad, rtol=0, atol=1e-5 * np.max(np.abs(forces)))


# --------------------------------------------------------------- short range
def test_short_range_known_answers_and_errors(pk):
    box = pk.BoxGeometry(100.0, 100.0, 10.0)
    s = pk.make_system([1.0, -1.0], np.ones(2), [[1.0, 1.0, 1.0], [4.0, 5.0, 1.0]], box)
    u, f = pk.short_range_energy_forces(s, box, 0.1, 40.0)
    assert u == pytest.approx(-erfc(0.5) / 5.0, rel=1e-13)
    np.testing.assert_allclose(f[0], -f[1], rtol=1e-14)
    empty = pk.make_system(np.zeros(0), np.zeros(0), np.zeros((0, 3)), box)
    u0, f0 = pk.short_range_energy_forces(empty, box, 1.0, 3.0)
    assert u0 == 0.0 and f0.shape == (0, 3)
    dup = pk.make_system([1.0, 1.0], np.ones(2), [[1, 1, 1], [1, 1, 1]], box)
    with pytest.raises(ValueError, match="coincident"):
        pk.short_range_energy_forces(dup, box, 1.0, 3.0)
    with pytest.raises(ValueError, match="half the in-plane"):
        pk.short_range_energy_forces(s, pk.BoxGeometry(10.0, 10.0, 10.0), 1.0, 5.5)


def test_short_range_dense_walls_matches_oracle(pk):
    # cfg3-like wall layers: ~10x mean density in thin z layers (load imbalance)
    from oracle import oracle as O
    from paper_2403_01521_b200.configs import make_workload
    wl = make_workload("cfg3")
    u, f = pk.short_range_energy_forces(wl.system, wl.box, wl.alpha, wl.params().r_c)
    g = load_golden("cfg3")
    assert u == pytest.approx(float(g["u_s_alone"]), rel=1e-10)
    idx = g["sample_idx"]
    np.testing.assert_allclose(f[idx], g["f_short"], rtol=0,
                               atol=1e-9 * np.max(np.abs(g["f_short"])))


# --------------------------------------------------------------- sampler
def test_sampler_statistics(pk):
    box = pk.BoxGeometry(100.0, 100.0, 10.0)
    smp = pk.ModeSampler(0.3, box, seed=11)
    n_draw = 20000
    rec = smp.batch_indices(n_draw)
    assert not np.any((rec[:, 0] == 0) & (rec[:, 1] == 0))
    assert smp.acceptance_rate > 0.9
    ax = smp.axx
    mmax = 30
    grid = np.arange(-mmax, mmax + 1)
    wx = np.exp(-(ax * grid) ** 2)
    weight = np.outer(wx, wx)
    weight[mmax, mmax] = 0.0
    counts = np.zeros_like(weight)
    inside = (np.abs(rec[:, 0]) <= mmax) & (np.abs(rec[:, 1]) <= mmax)
    np.add.at(counts, (rec[inside, 0] + mmax, rec[inside, 1] + mmax), 1.0)
    expected = n_draw * weight / weight.sum()
    keep = expected >= 5.0
    obs = np.append(counts[keep], n_draw - counts[keep].sum())
    exp = np.append(expected[keep], n_draw - expected[keep].sum())
    _, p = chisquare(obs, exp * obs.sum() / exp.sum())
    assert p > 1e-3
    # the reference chain's own draws (different RNG stream, same law): a
    # two-sample chi-square test on the joint (mx, my) histogram -- pooled bins
    # with >= 10 expected draws per sample, the rest merged into one bin -- and
    # the same acceptance rate
    from scipy.stats import chi2_contingency
    g = load_golden("units")
    ref = g["sampler_idx_a03_L100_seed11"]
    keys = lambda a: (a[:, 0].astype(np.int64) + 1000) * 4000 + (a[:, 1].astype(np.int64) + 1000)
    ka, kb = keys(rec), keys(ref)
    cells, pooled = np.unique(np.concatenate([ka, kb]), return_counts=True)
    big = cells[pooled >= 20]
    ca = np.array([np.sum(ka == c) for c in big] + [np.sum(~np.isin(ka, big))])
    cb = np.array([np.sum(kb == c) for c in big] + [np.sum(~np.isin(kb, big))])
    _, p2, _, _ = chi2_contingency(np.vstack([ca, cb]))
    assert p2 > 1e-3, p2
    assert len(big) > 50
    assert abs(smp.acceptance_rate - float(g["sampler_acc_a03_L100_seed11"])) < 0.02


def test_sampler_determinism_and_scaling(pk):
    box = pk.BoxGeometry(80.0, 120.0, 10.0)
    a = pk.ModeSampler(0.25, box, seed=4).batch_indices(300)
    b = pk.ModeSampler(0.25, box, seed=4).batch_indices(300)
    c = pk.ModeSampler(0.25, box, seed=5).batch_indices(300)
    np.testing.assert_array_equal(a, b)
    assert np.any(a != c)
    kb = pk.ModeSampler(0.25, box, seed=4).batch(300)
    np.testing.assert_array_equal(kb[:, 0], 2 * np.pi * a[:, 0] / box.lx)
    np.testing.assert_array_equal(kb[:, 1], 2 * np.pi * a[:, 1] / box.ly)
    np.testing.assert_array_equal(kb[:, 2], np.hypot(kb[:, 0], kb[:, 1]))
    with pytest.raises(ValueError, match="thin"):
        pk.ModeSampler(0.3, box, thin=0)
    with pytest.raises(ValueError, match="batch size"):
        pk.metropolis_batch(pk.ModeSampler(0.3, box, seed=5), 0)


def test_rb_estimator_unbiased_and_variance_scaling(pk):
    box = pk.BoxGeometry(10.0, 10.0, 5.0)
    s = _slab_system(pk, 25, box, 61)
    params = pk.make_ewald_params(0.8, 4.0, box)
    soe8 = pk.build_soe_contour(8)
    est = pk.run_many_batches(s, box, params, soe8, n_batches=3000, P=16, seed=2)
    truth = pk.total_energy_soe(s, box, params, soe8).total
    d = pk.variance_diagnostics(est)
    assert abs(d["mean"] - truth) <= 3.0 * d["stderr"]
    s2 = _slab_system(pk, 25, box, 62)
    e16 = pk.run_many_batches(s2, box, params, soe8, n_batches=4000, P=16, seed=3)
    e64 = pk.run_many_batches(s2, box, params, soe8, n_batches=4000, P=64, seed=4)
    ratio = np.var(e64, ddof=1) / np.var(e16, ddof=1)
    assert 0.2 <= ratio <= 0.32


def test_single_particle_rb_estimate_is_charge_constant(pk):
    box = pk.BoxGeometry(10.0, 10.0, 5.0)
    s = pk.make_system([1.0], [1.0], [[2.0, 3.0, 2.5]], box)
    import warnings
    with warnings.catch_warnings():
        warnings.simplefilter("ignore")
        H = pk.normalization_H(0.8, box)
    c_q = pk.charge_term_sum(0.8, box, 1.0)
    smp = pk.ModeSampler(0.8, box, seed=6)
    soe8 = pk.build_soe_contour(8)
    assert all(pk.rb_energy_estimate(s, box, 0.8, soe8, smp.batch(16), H) == c_q
               for _ in range(3))


@pytest.mark.parametrize("bad", [np.nan, np.inf, -np.inf])
def test_nonfinite_z_rejected_by_device_status(pk, bad):
    """core.py:206-207 via the device status word (no host scan on the eval path)."""
    box = pk.BoxGeometry(10.0, 10.0, 5.0)
    s = _slab_system(pk, 20, box, 71)
    pos = s.pos.copy()
    pos[7, 2] = bad
    s = pk.make_system(s.charge, np.ones(s.n), pos)  # no box: make_system would reject inf
    params = pk.make_ewald_params(0.8, 4.0, box)
    soe8 = pk.build_soe_contour(8)
    smp = pk.ModeSampler(0.8, box, seed=1)
    with pytest.raises(ValueError, match="finite"):
        pk.rb_energy_forces(s, box, params, soe8, smp, 8)
    with pytest.raises(ValueError, match="finite"):
        pk.soe_energy_forces(s, box, params, soe8)
    # the context recovers (status word reset per evaluation)
    good = _slab_system(pk, 20, box, 71)
    pk.soe_energy_forces(good, box, params, soe8)


def test_device_sampler_handover_and_host_buffers(pk):
    """rb_energy_forces with a ModeSampler takes the k-set on device
    (batch_device) and evaluates through slab_evaluate_host; a twin sampler's
    host batch(P) through the stub path and the device-buffer evaluate agree,
    for pageable and page-locked inputs, and the chain state advances alike."""
    from paper_2403_01521_b200.engine import pinned_like
    box = pk.BoxGeometry(14.0, 14.0, 7.0)
    s = _slab_system(pk, 3000, box, 5)
    params = pk.make_ewald_params(0.7, 3.0, box)
    soe8 = pk.build_soe_contour(8)
    H = pk.normalization_H(0.7, box)
    a, b = pk.ModeSampler(0.7, box, seed=9), pk.ModeSampler(0.7, box, seed=9)

    class Stub:
        def __init__(self, m):
            self.m = m

        def batch(self, P):
            return self.m

    for pinned in (False, True):
        sys_ = s
        if pinned:
            sys_ = pk.make_system(s.charge, s.mass, s.pos, box)
            sys_.pos, sys_.charge = pinned_like(s.pos), pinned_like(s.charge)
        bd1, f1 = pk.rb_energy_forces(sys_, box, params, soe8, a, 12, H=H, c_q=0.0)
        modes = b.batch(12)
        bd2, f2 = pk.rb_energy_forces(s, box, params, soe8, Stub(modes), 12, H=H, c_q=0.0)
        assert bd1.total == pytest.approx(bd2.total, rel=1e-12, abs=1e-12)
        np.testing.assert_allclose(f1, f2, rtol=0, atol=1e-12 * np.max(np.abs(f2)))
    assert a.accepted == b.accepted and a.steps == b.steps
    # the device-buffer entry (slab_evaluate) on the same k-set
    from paper_2403_01521_b200.engine import get_engine, to_device
    eng = get_engine()
    cv = (H / 12) * (2 / np.sqrt(np.pi)) * 0.7
    e_d, f_d = eng.evaluate(to_device(s.pos), to_device(s.charge), box, 0.7, params.r_c, soe8,
                            to_device(modes), cv, 0.0)
    e_d = e_d.cpu().numpy()
    assert float(e_d[0] + e_d[1] + e_d[2] - e_d[3] + e_d[4]) == pytest.approx(bd2.total,
                                                                            rel=1e-12)
    np.testing.assert_array_equal(f_d.cpu().numpy(), f2)


# --------------------------------------------------------------- device evaluator
def test_graph_replay_and_shard_sum_equal_single_eval(pk):
    import torch
    from paper_2403_01521_b200.configs import make_workload
    from paper_2403_01521_b200.engine import DeviceEvaluator
    wl = make_workload("small_2000")
    soe = pk.build_soe_contour(wl.m)
    g = load_golden("small_2000")
    kw = dict(P=wl.P, H=float(g["H"]), c_q=float(g["c_q"]), modes=g["modes"])
    ev = DeviceEvaluator(wl.system, wl.box, wl.params(), soe, **kw)
    ev.step()
    e1, f1 = ev.energy.clone(), ev.forces.clone()
    ev.capture()
    ev.step()
    torch.cuda.synchronize()
    assert torch.equal(e1, ev.energy) and torch.equal(f1, ev.forces)
    # two shards evaluated one after the other on this GPU, summed by hand
    tot = torch.zeros_like(ev.packed)
    for r in range(2):
        evr = DeviceEvaluator(wl.system, wl.box, wl.params(), soe, rank=r, world=1, **kw)
        evr.rank, evr.world, evr.reduce = r, 2, False   # shard, no collective
        from paper_2403_01521_b200.sharding import mode_slice
        evr.t0, evr.t1 = mode_slice(evr.P, r, 2)
        evr.step()
        tot += evr.packed
    torch.cuda.synchronize()
    e, f = tot[3 * wl.n:].cpu().numpy(), tot[:3 * wl.n].view(wl.n, 3).cpu().numpy()
    for val, key in zip(e, ("u_s", "u_l_k", "u_l_0", "u_self", "u_ps")):
        assert val == pytest.approx(float(g[key]), rel=1e-10), key
    np.testing.assert_allclose(f, g["forces"], rtol=0, atol=1e-9 * float(g["fmax"]))


def test_scan_event_graph_times_the_scan_and_matches_the_step(pk):
    """bench.py's roofline graph: the step captured with the scan's timing events
    as external record nodes stamps a positive scan span on every replay, inside
    the full step, and computes the same bits as the step's own graph."""
    import torch
    from paper_2403_01521_b200.configs import make_workload
    from paper_2403_01521_b200.engine import DeviceEvaluator
    wl = make_workload("small_2000")
    soe = pk.build_soe_contour(wl.m)
    g = load_golden("small_2000")
    ev = DeviceEvaluator(wl.system, wl.box, wl.params(), soe, P=wl.P, H=float(g["H"]),
                         c_q=float(g["c_q"]), modes=g["modes"])
    ev.capture()
    ev.step()
    torch.cuda.synchronize()
    e1, f1 = ev.energy.clone(), ev.forces.clone()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s, t = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()  # materialise the cudaEvent_t handles (torch creates them lazily)
    b.record()
    torch.cuda.synchronize()
    gt = ev.capture(scan_events=(a, b))
    assert ev.graph is not gt  # the step's own graph is kept
    spans = []
    for _ in range(3):
        s.record()
        gt.replay()
        t.record()
        torch.cuda.synchronize()
        spans.append((a.elapsed_time(b), s.elapsed_time(t)))
    for scan, step in spans:
        assert 0.0 < scan <= step
    assert torch.equal(e1, ev.energy) and torch.equal(f1, ev.forces)


def test_run_many_batches_matches_per_batch_estimates(pk):
    """Batched forward-sweep energies (slab_batch_energies, several device passes)
    equal one rb_energy_estimate per batch plus the deterministic terms.  Like the
    reference (rbse2d.py:346), all n_batches * P modes come from ONE sampler call
    (chain draws are not invariant under re-batching, there or here)."""
    box = pk.BoxGeometry(10.0, 10.0, 5.0)
    s = _slab_system(pk, 25, box, 63)
    params = pk.make_ewald_params(0.8, 4.0, box)
    soe8 = pk.build_soe_contour(8)
    _batches_vs_estimates(pk, s, box, params, soe8, 16, 600)  # three 4096-mode passes
    # P = 12: passes of 341 batches (4092 items: a partial warp) and a 59-batch
    # tail (708 items = 22 warps + 4 items in the remainder sweep)
    _batches_vs_estimates(pk, s, box, params, soe8, 12, 400)


def _batches_vs_estimates(pk, s, box, params, soe8, P, nb):
    est = pk.run_many_batches(s, box, params, soe8, n_batches=nb, P=P, seed=21)
    H = pk.normalization_H(0.8, box)
    c_q = pk.charge_term_sum(0.8, box, float(np.sum(s.charge ** 2)))
    bd, _ = pk.soe_energy_forces(s, box, params, soe8)
    det = bd.u_s + bd.u_l_0 - bd.u_self + bd.u_ps
    allm = pk.ModeSampler(0.8, box, seed=21).batch(nb * P)
    for b in range(nb):
        modes = allm[b * P:(b + 1) * P]
        if b % 97 == 0 or b == nb - 1:
            want = pk.rb_energy_estimate(s, box, 0.8, soe8, modes, H, c_q) + det
            assert est[b] == pytest.approx(want, rel=1e-12, abs=1e-12), b


@pytest.mark.parametrize("W,forces", [(3, True), (4, False), (2, True)])
def test_zsplit_ranks_sum_to_the_single_gpu_evaluation(pk, W, forces):
    """z-split multi-GPU decomposition (SURVEY 8(e) alternative), emulated on one
    GPU with one context per rank: phase 1 on every rank, the all-gather as a
    concatenation, phase 2 on every rank; summed forces / energies equal the
    single-GPU evaluation."""
    import torch
    from paper_2403_01521_b200 import _native
    from paper_2403_01521_b200.configs import make_workload
    from paper_2403_01521_b200.engine import Engine, get_engine
    wl = make_workload("small_2000")
    soe = pk.build_soe_contour(wl.m)
    params = wl.params()
    eng = get_engine()
    dev = eng.device
    pos = torch.as_tensor(wl.system.pos).to(dev)
    q = torch.as_tensor(wl.system.charge).to(dev)
    smp = pk.ModeSampler(wl.alpha, wl.box, seed=3)
    modes = torch.as_tensor(smp.batch(wl.P)).to(dev)
    args = (pos, q, wl.box, wl.alpha, params.r_c, soe, modes, 0.37, 1.5)
    e1, f1 = eng.evaluate(*args, want_forces=forces)
    e1 = e1.cpu().numpy()
    cnt = int(_native.load().slab_zsplit_exchange_doubles(wl.P, wl.m, 1 if forces else 0))
    engines = [Engine(dev) for _ in range(W)]
    xloc = [torch.zeros(cnt, dtype=torch.float64, device=dev) for _ in range(W)]
    for r in range(W):
        engines[r].evaluate(*args, want_forces=forces, shard=(r, W), shard_mode=1, phase=1,
                            xchg=xloc[r])
    xall = torch.cat(xloc)
    etot = np.zeros(8)
    ftot = np.zeros((wl.n, 3))
    for r in range(W):
        e, f = engines[r].evaluate(*args, want_forces=forces, shard=(r, W), shard_mode=1,
                                   phase=2, xchg=xall)
        e = e.cpu().numpy()
        assert int(e[5]) == 0
        etot[:5] += e[:5]
        if forces:
            ftot += f.cpu().numpy()
    for k in range(5):
        assert etot[k] == pytest.approx(e1[k], rel=1e-12, abs=1e-12), k
    if forces:
        f1 = f1.cpu().numpy()
        np.testing.assert_allclose(ftot, f1, rtol=0, atol=1e-12 * np.max(np.abs(f1)))


@pytest.mark.parametrize("tag,box_l,alpha,s_par", [("a", (10.0, 10.0, 5.0), 0.6, 3.0),
                                                   ("b", (14.0, 11.0, 7.0), 0.8, 3.5)])
def test_ewald2d_reference_solver_matches_reference(pk, tag, box_l, alpha, s_par):
    """the O(N^2 K) Ewald2D reference on device against the
    reference's own ref_energy_forces (stable), the naive xi variant and the
    k = 0 mode (tests/golden/ewald_ref.npz); and SOEwald2D agrees with it to the
    SOE accuracy (M = 16, eps ~ 1e-9)."""
    g = load_golden("ewald_ref")
    box = pk.BoxGeometry(*box_l)
    pos = g[f"{tag}_pos"]
    n = len(pos)
    s = pk.make_system(np.where(np.arange(n) % 2 == 0, 1.0, -1.0), np.ones(n), pos, box)
    params = pk.make_ewald_params(alpha, s_par, box)
    bd, f = pk.ref_energy_forces(s, box, params)
    for k in ("u_s", "u_l_k", "u_l_0", "u_self", "u_ps"):
        ref = float(g[f"{tag}_{k}"])
        assert getattr(bd, k) == pytest.approx(ref, rel=1e-10, abs=1e-12), k
    fref = g[f"{tag}_forces"]
    np.testing.assert_allclose(f, fref, rtol=0, atol=1e-9 * np.max(np.abs(fref)))
    un, fn = pk.fourier_energy_forces_ref(s, box, params, "naive")
    assert un == pytest.approx(float(g[f"{tag}_naive_u"]), rel=1e-10)
    np.testing.assert_allclose(fn, g[f"{tag}_naive_f"], rtol=0,
                               atol=1e-9 * np.max(np.abs(g[f"{tag}_naive_f"])))
    u0, f0 = pk.zero_mode_energy_forces_ref(s, box, alpha)
    assert u0 == pytest.approx(float(g[f"{tag}_zero_u"]), rel=1e-10)
    np.testing.assert_allclose(f0, g[f"{tag}_zero_f"], rtol=0,
                               atol=1e-9 * np.max(np.abs(g[f"{tag}_zero_f"])))
    soe = pk.build_soe_contour(16)
    bs, fs = pk.soe_energy_forces(s, box, params, soe)
    assert bs.total == pytest.approx(bd.total, rel=1e-7)
    with pytest.raises(ValueError, match="neutral"):
        pk.ref_energy_forces(pk.make_system(np.ones(n), np.ones(n), pos, box), box, params)


def test_batch_energies_match_reference_batches(pk):
    """SURVEY 8(f) rank 2 pinned to the REAL reference: the per-batch energies of
    rbse2d.py:320-363 (_rb_batch_energy_kernel, k-sequence from the reference
    sampler injected; tests/golden/batches.npz) against slab_batch_energies --
    N = 1e4, P = 100, 41 batches = a 40-batch device pass plus a 1-batch tail
    pass with its own plan -- and the deterministic part u_det."""
    import torch
    from paper_2403_01521_b200.configs import make_workload
    from paper_2403_01521_b200.engine import get_engine
    from paper_2403_01521_b200.rbse2d import _rb_commonv
    g = load_golden("batches")
    wl = make_workload("cfg5_1e4")
    soe = pk.build_soe_contour(wl.m)
    params = wl.params()
    eng = get_engine()
    d = lambda a: torch.as_tensor(np.ascontiguousarray(a)).to(eng.device)
    P, nb = int(g["P"]), int(g["n_batches"])
    out, status = eng.batch_energies(d(wl.system.pos), d(wl.system.charge), soe, wl.alpha,
                                     wl.box.area, d(g["modes"]), nb, P,
                                     _rb_commonv(float(g["H"]), P, wl.alpha))
    assert int(status.cpu().item()) == 0
    got = out.cpu().numpy()
    scale = np.max(np.abs(g["batch_u"]))
    assert np.max(np.abs(got - g["batch_u"])) <= 1e-10 * scale
    bd, _ = pk.soe_energy_forces(wl.system, wl.box, params, soe)
    u_det = bd.u_s + bd.u_l_0 - bd.u_self + bd.u_ps + float(g["c_q"])
    assert u_det == pytest.approx(float(g["u_det"]), rel=1e-10)
