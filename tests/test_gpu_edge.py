"""GPU: edge cases and size-independent properties of the evaluation.

Small / ragged cases are checked against the CPU oracle (oracle/, itself pinned
to the reference's goldens in test_oracle.py); at N = 1e7 -- beyond what the
oracle or the reference finish in test time -- size-independent identities
(charge scaling, translation invariance, Newton's third law, shard sums)."""

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

E_TOL = 1e-10
F_TOL = 1e-9


@pytest.fixture(scope="module")
def pk():
    import paper_2403_01521_b200 as pk
    return pk


def _oracle_eval(pk, s, box, params, soe, modes, cv, cq):
    from oracle import oracle as O
    O.build()
    e, f, flag = O.energy_forces(s.pos, s.charge, box, params.alpha, params.r_c, modes,
                                 np.broadcast_to(cv, (len(modes),)).copy(), cq, soe.w, soe.s)
    assert flag == 0
    return e, f


def _check(bd, f, e_ref, f_ref):
    got = [bd.u_s, bd.u_l_k, bd.u_l_0, bd.u_self, bd.u_ps]
    for g, r in zip(got, e_ref):
        assert abs(g - r) <= E_TOL * max(abs(r), 1e-300) or g == r == 0
    if f_ref.size:
        fmax = max(np.max(np.abs(f_ref)), 1e-300)
        assert np.max(np.abs(f - f_ref)) <= F_TOL * fmax


class _Stub:
    def __init__(self, modes):
        self.modes = modes

    def batch(self, P):
        return self.modes


@pytest.mark.parametrize("n", [0, 1, 2, 3, 17, 257, 4097])
def test_ragged_sizes_match_oracle(pk, n):
    """Empty, single, tiny and chunk-ragged systems (chunk lengths are powers of
    two; 257 and 4097 leave one-particle tail chunks), charged slab walls."""
    rng = np.random.default_rng(100 + n)
    box = pk.BoxGeometry(12.0, 9.0, 7.0, sigma_top=0.004, sigma_bot=-0.0015)
    pos = rng.uniform([0, 0, 0.1], [12.0, 9.0, 6.9], size=(n, 3))
    q = rng.choice([-1.0, 1.0, 2.0], size=n)
    s = pk.make_system(q, np.ones(n), pos, box)
    params = pk.make_ewald_params(0.9, 3.5, box)
    soe = pk.build_soe_contour(16)
    modes = pk.ModeSampler(0.9, box, seed=n).batch(13)
    H = pk.normalization_H(0.9, box)
    cq = pk.charge_term_sum(0.9, box, float(np.sum(q ** 2)))
    bd, f = pk.rb_energy_forces(s, box, params, soe, _Stub(modes), 13, H=H, c_q=cq)
    assert f.shape == (n, 3)
    cv = (H / 13) * (2 / np.sqrt(np.pi)) * 0.9
    e_ref, f_ref = _oracle_eval(pk, s, box, params, soe, modes, cv, cq)
    _check(bd, f, e_ref, f_ref)


@pytest.mark.parametrize("P", [15, 16, 17, 20, 24, 36, 100])
@pytest.mark.parametrize("M", [16, 24])
def test_mode_counts_and_warp_layouts_match_oracle(pk, P, M):
    """Sweep layouts by mode count: a force plan's warp holds 16 modes x 2
    directions, so P = 15 / 24 leave a partial warp, 16 is exact, and 17 / 20 /
    36 / 100 send their leftover modes (P mod 16 <= 4) to the remainder sweep;
    M = 24 (12 pairs) takes the one-CTA-per-SM form.  n = 3000 spans several
    chunks of both sweeps."""
    rng = np.random.default_rng(P * 100 + M)
    box = pk.BoxGeometry(20.0, 20.0, 10.0, sigma_top=0.002, sigma_bot=-0.001)
    n = 3000
    pos = rng.uniform([0, 0, 0.1], [20.0, 20.0, 9.9], size=(n, 3))
    q = rng.choice([-1.0, 1.0, 2.0], size=n)
    s = pk.make_system(q, np.ones(n), pos, box)
    params = pk.make_ewald_params(0.8, 3.6, box)
    soe = pk.build_soe_contour(M)
    modes = pk.ModeSampler(0.8, box, seed=P).batch(P)
    H = pk.normalization_H(0.8, box)
    cq = pk.charge_term_sum(0.8, box, float(np.sum(q ** 2)))
    bd, f = pk.rb_energy_forces(s, box, params, soe, _Stub(modes), P, H=H, c_q=cq)
    cv = (H / P) * (2 / np.sqrt(np.pi)) * 0.8
    e_ref, f_ref = _oracle_eval(pk, s, box, params, soe, modes, cv, cq)
    _check(bd, f, e_ref, f_ref)
    # energy-only plans (forward items only, 32 consecutive items per warp)
    from paper_2403_01521_b200 import rbse2d
    u = rbse2d.rb_energy_estimate(s, box, 0.8, soe, modes, H, c_q=cq)
    assert abs(u - e_ref[1]) <= E_TOL * abs(e_ref[1])


@pytest.mark.parametrize("M", [4, 6, 10, 12, 14, 18, 20, 22])
def test_every_soe_term_count_matches_oracle(pk, M):
    """Each sweep / aggregate / k = 0 instantiation (2 .. 11 conjugate pairs; 8
    and 12 are covered above): energies and forces against the oracle, P = 20
    (remainder groups) and P = 9 (a partial warp), n spanning several chunks."""
    rng = np.random.default_rng(M)
    box = pk.BoxGeometry(18.0, 16.0, 9.0, sigma_top=-0.003, sigma_bot=0.002)
    n = 1500
    pos = rng.uniform([0, 0, 0.05], [18.0, 16.0, 8.95], size=(n, 3))
    q = rng.choice([-1.0, 1.0, 2.0], size=n)
    s = pk.make_system(q, np.ones(n), pos, box)
    params = pk.make_ewald_params(0.8, 3.6, box)
    soe = pk.build_soe_contour(M)
    H = pk.normalization_H(0.8, box)
    cq = pk.charge_term_sum(0.8, box, float(np.sum(q ** 2)))
    for P in (20, 9):
        modes = pk.ModeSampler(0.8, box, seed=M + P).batch(P)
        bd, f = pk.rb_energy_forces(s, box, params, soe, _Stub(modes), P, H=H, c_q=cq)
        cv = (H / P) * (2 / np.sqrt(np.pi)) * 0.8
        e_ref, f_ref = _oracle_eval(pk, s, box, params, soe, modes, cv, cq)
        _check(bd, f, e_ref, f_ref)


def test_single_mode_and_full_sum_small(pk):
    """P = 1 (one item pair per chunk) and a full deterministic mode sum."""
    rng = np.random.default_rng(7)
    box = pk.BoxGeometry(15.0, 15.0, 6.0)
    n = 600
    s = pk.make_system(np.where(np.arange(n) % 2 == 0, 1.0, -1.0), np.ones(n),
                       rng.uniform([0, 0, 0.2], [15, 15, 5.8], size=(n, 3)), box)
    params = pk.make_ewald_params(0.7, 3.0, box)
    soe = pk.build_soe_contour(8)
    modes = pk.ModeSampler(0.7, box, seed=1).batch(1)
    H = pk.normalization_H(0.7, box)
    bd, f = pk.rb_energy_forces(s, box, params, soe, _Stub(modes), 1, H=H, c_q=0.0)
    e_ref, f_ref = _oracle_eval(pk, s, box, params, soe, modes,
                                H * (2 / np.sqrt(np.pi)) * 0.7, 0.0)
    _check(bd, f, e_ref, f_ref)


def test_boundary_heights_and_z_ties_match_oracle(pk):
    """Particles exactly on both walls (z = 0, z = Lz, -0.0), whole layers of
    equal z (ties resolved by input order, like the reference's stable sort)
    and charged walls: energies, forces and the permutation against the
    oracle."""
    rng = np.random.default_rng(44)
    box = pk.BoxGeometry(14.0, 14.0, 6.0, sigma_top=0.002, sigma_bot=-0.001)
    n = 1200
    pos = rng.uniform([0, 0, 0], [14.0, 14.0, 6.0], size=(n, 3))
    pos[:40, 2] = 0.0
    pos[40:60, 2] = -0.0
    pos[60:100, 2] = 6.0
    pos[100:400, 2] = np.repeat(rng.uniform(0.5, 5.5, 30), 10)  # 30 layers of 10
    q = np.where(np.arange(n) % 2 == 0, 1.0, -1.0)
    s = pk.make_system(q, np.ones(n), pos, box)
    perm = pk.sort_by_z(s, box.lz)
    np.testing.assert_array_equal(perm, np.argsort(s.pos[:, 2], kind="stable"))
    params = pk.make_ewald_params(0.8, 3.2, box)
    soe = pk.build_soe_contour(16)
    modes = pk.ModeSampler(0.8, box, seed=8).batch(9)
    H = pk.normalization_H(0.8, box)
    cq = pk.charge_term_sum(0.8, box, float(np.sum(q ** 2)))
    bd, f = pk.rb_energy_forces(s, box, params, soe, _Stub(modes), 9, H=H, c_q=cq)
    e_ref, f_ref = _oracle_eval(pk, s, box, params, soe, modes,
                                (H / 9) * (2 / np.sqrt(np.pi)) * 0.8, cq)
    _check(bd, f, e_ref, f_ref)


@pytest.mark.parametrize("table", ["real_m1", "shuffled_plus_real"])
def test_real_and_unordered_soe_tables_match_oracle(pk, table):
    """Tables beyond the built contours: the single real-exponent term of the
    reference's soe tests (w = 1, s = 2), and a built 8-term table in shuffled
    order plus a real term -- every term real or with its conjugate somewhere;
    a complex term without its conjugate is rejected."""
    rng = np.random.default_rng(21)
    box = pk.BoxGeometry(15.0, 15.0, 6.0)
    n = 900
    s = pk.make_system(np.where(np.arange(n) % 2 == 0, 1.0, -1.0), np.ones(n),
                       rng.uniform([0, 0, 0.2], [15, 15, 5.8], size=(n, 3)), box)
    alpha = 0.9
    params = pk.make_ewald_params(alpha, 3.0, box)
    if table == "real_m1":
        w, sv = np.array([1.0 + 0j]), np.array([2.0 + 0j])
    else:
        b8 = pk.build_soe_contour(8)
        order = rng.permutation(8)
        w = np.concatenate([b8.w[order], [0.25 + 0j]])
        sv = np.concatenate([b8.s[order], [3.5 + 0j]])
    soe = pk.SOEApprox(m=len(w), w=w, s=sv, eps_certified=1.0, domain_max=20.0)
    modes = pk.ModeSampler(alpha, box, seed=2).batch(7)
    H = pk.normalization_H(alpha, box)
    bd, f = pk.rb_energy_forces(s, box, params, soe, _Stub(modes), 7, H=H, c_q=0.0)
    e_ref, f_ref = _oracle_eval(pk, s, box, params, soe, modes,
                                (H / 7) * (2 / np.sqrt(np.pi)) * alpha, 0.0)
    _check(bd, f, e_ref, f_ref)


@pytest.mark.parametrize("table", ["lone_plus_real", "contour_halves", "all_lone"])
def test_lone_complex_soe_terms_match_oracle(pk, table):
    """Tables with complex terms that have NO conjugate partner (the reference's
    sweep takes any (w, s); load_soe_table reads any table): each lone term runs
    as a half-weight pair plus a second, input-swapped pass (capi.cu
    prepare_soe).  RB and full-mode-sum evaluations (energies, forces, k = 0
    mode) and the batched energies against the oracle, which restates the
    reference's per-term loops."""
    rng = np.random.default_rng(31)
    box = pk.BoxGeometry(15.0, 15.0, 6.0)
    n = 700
    s = pk.make_system(np.where(np.arange(n) % 2 == 0, 1.0, -1.0), np.ones(n),
                       rng.uniform([0, 0, 0.2], [15, 15, 5.8], size=(n, 3)), box)
    alpha = 0.9
    params = pk.make_ewald_params(alpha, 3.0, box)
    if table == "lone_plus_real":
        w = np.array([1.0 + 0.5j, 1.0 + 0j])
        sv = np.array([2.0 + 1j, 3.0 + 0j])
    elif table == "contour_halves":   # a built table with two conjugates dropped
        b8 = pk.build_soe_contour(8)
        keep = [0, 1, 2, 3, 4, 6]           # terms 7 and 5 (partners of 0 and 2) removed
        order = rng.permutation(len(keep))
        w, sv = b8.w[keep][order], b8.s[keep][order]
    else:
        w = np.array([0.7 - 0.2j, 0.3 + 0.9j, 1.1 + 0.1j])
        sv = np.array([1.5 + 0.8j, 2.5 - 1.7j, 0.9 + 3.0j])
    soe = pk.SOEApprox(m=len(w), w=w, s=sv, eps_certified=1.0, domain_max=20.0)
    modes = pk.ModeSampler(alpha, box, seed=4).batch(9)
    H = pk.normalization_H(alpha, box)
    cv = (H / 9) * (2 / np.sqrt(np.pi)) * alpha
    bd, f = pk.rb_energy_forces(s, box, params, soe, _Stub(modes), 9, H=H, c_q=0.0)
    e_ref, f_ref = _oracle_eval(pk, s, box, params, soe, modes, cv, 0.0)
    _check(bd, f, e_ref, f_ref)
    # the deterministic full mode sum through the same two passes
    from paper_2403_01521_b200.soewald2d import full_sum_constants
    cvf, uq = full_sum_constants(params, box, float(np.sum(s.charge ** 2)))
    bdf, ff = pk.soe_energy_forces(s, box, params, soe)
    e_reff, f_reff = _oracle_eval(pk, s, box, params, soe, params.kmodes, cvf, uq)
    _check(bdf, ff, e_reff, f_reff)
    # batched energies: every batch's forward sweep (one device pass + the lone pass)
    import torch
    from oracle import oracle as O
    from paper_2403_01521_b200.engine import get_engine
    eng = get_engine()
    allm = pk.ModeSampler(alpha, box, seed=5).batch(5 * 9)
    d = lambda a: torch.as_tensor(np.ascontiguousarray(a)).to(eng.device)
    out, status = eng.batch_energies(d(s.pos), d(s.charge), soe, alpha, box.area, d(allm), 5, 9, cv)
    got = out.cpu().numpy()
    perm = O.sort_perm(s.pos[:, 2], box.lz)
    xs, ys, zs = (np.ascontiguousarray(s.pos[perm, i]) for i in range(3))
    for b in range(5):
        u, _ = O.fourier_sweep(xs, ys, zs, s.charge[perm], allm[b * 9:(b + 1) * 9],
                               np.full(9, cv), soe.w, soe.s, alpha, box.area)
        assert abs(got[b] - u) <= E_TOL * max(abs(u), 1e-300), b


@pytest.mark.parametrize("table", ["real_m1", "pairs_plus_real"])
def test_singular_soe_terms_match_oracle(pk, table):
    """A mode with |k| within 2e-6 k of a real exponent alpha*s_l takes the
    reference's analytic-limit branch (soewald2d.py:116-124: c_l = 0, the term's
    weight through the extra h chain); checked against the oracle, which
    restates that branch, with forces (both directions) and energies."""
    rng = np.random.default_rng(33)
    box = pk.BoxGeometry(12.0, 12.0, 6.0)
    n = 700
    s = pk.make_system(np.where(np.arange(n) % 2 == 0, 1.0, -1.0), np.ones(n),
                       rng.uniform([0, 0, 0.2], [12, 12, 5.8], size=(n, 3)), box)
    alpha = 0.9
    params = pk.make_ewald_params(alpha, 3.0, box)
    if table == "real_m1":
        w, sv = np.array([1.0 + 0j]), np.array([2.0 + 0j])
        kc = alpha * 2.0
    else:
        b8 = pk.build_soe_contour(8)
        w = np.concatenate([b8.w, [0.25 + 0j]])
        sv = np.concatenate([b8.s, [3.5 + 0j]])
        kc = alpha * 3.5
    soe = pk.SOEApprox(m=len(w), w=w, s=sv, eps_certified=1.0, domain_max=20.0)
    other = pk.ModeSampler(alpha, box, seed=5).batch(5)
    ks = kc * (1.0 + 3e-7)  # singular: |alpha s - k| < 2e-6 k
    sing = np.array([[ks * 0.6, ks * 0.8, ks], [-ks, 0.0, ks]])
    modes = np.vstack([other[:2], sing, other[2:]])
    P = len(modes)
    H = pk.normalization_H(alpha, box)
    bd, f = pk.rb_energy_forces(s, box, params, soe, _Stub(modes), P, H=H, c_q=0.0)
    e_ref, f_ref = _oracle_eval(pk, s, box, params, soe, modes,
                                (H / P) * (2 / np.sqrt(np.pi)) * alpha, 0.0)
    _check(bd, f, e_ref, f_ref)


@pytest.mark.parametrize("name", ["cfg3", "cfg4"])
def test_run_to_run_bit_reproducible(pk, name):
    """Fixed-order sums everywhere (no atomics on values), also with the short
    range, the k = 0 chain and the sampler on their own streams: two
    evaluations of the same input are bit-identical, through the host-buffer
    entry and the device-resident evaluator."""
    import torch
    from paper_2403_01521_b200.configs import make_workload
    from paper_2403_01521_b200.engine import DeviceEvaluator
    wl = make_workload(name)
    soe = pk.build_soe_contour(wl.m)
    params = wl.params()
    modes = pk.ModeSampler(wl.alpha, wl.box, seed=4).batch(wl.P)
    H = pk.normalization_H(wl.alpha, wl.box)
    runs = [pk.rb_energy_forces(wl.system, wl.box, params, soe, _Stub(modes), wl.P, H=H,
                                c_q=0.0) for _ in range(2)]
    assert runs[0][0] == runs[1][0]
    np.testing.assert_array_equal(runs[0][1], runs[1][1])
    outs = []
    for _ in range(2):
        ev = DeviceEvaluator(wl.system, wl.box, params, soe, P=wl.P, H=H, c_q=0.0, seed=11)
        ev.step()
        ev.step()
        torch.cuda.synchronize()
        outs.append((ev.energy.cpu().numpy().copy(), ev.forces.cpu().numpy().copy()))
        del ev
    np.testing.assert_array_equal(outs[0][0], outs[1][0])
    np.testing.assert_array_equal(outs[0][1], outs[1][1])


@pytest.mark.parametrize("n", [30000, 60000])
def test_pair_row_split_sizes_match_oracle(pk, n):
    """Home counts below one resident wave of threads split each neighbour row
    over 4 (n = 3e4) or 2 (n = 6e4) lanes combined by a shuffle tree."""
    rng = np.random.default_rng(n)
    L = (2 * n / 0.1) ** (1 / 3)
    box = pk.BoxGeometry(L, L, L / 2)
    pos = rng.uniform([0, 0, 0.05], [L, L, L / 2 - 0.05], size=(n, 3))
    q = np.where(np.arange(n) % 2 == 0, 1.0, -1.0)
    s = pk.make_system(q, np.ones(n), pos, box)
    alpha = 0.4
    params = pk.make_ewald_params(alpha, 3.0, box)
    soe = pk.build_soe_contour(8)
    modes = pk.ModeSampler(alpha, box, seed=n).batch(5)
    H = pk.normalization_H(alpha, box)
    bd, f = pk.rb_energy_forces(s, box, params, soe, _Stub(modes), 5, H=H, c_q=0.0)
    e_ref, f_ref = _oracle_eval(pk, s, box, params, soe, modes,
                                (H / 5) * (2 / np.sqrt(np.pi)) * alpha, 0.0)
    _check(bd, f, e_ref, f_ref)


@pytest.mark.parametrize("box_xy", [15.0, 11.0])
def test_alpha_rc_beyond_erfcx_table(pk, box_xy):
    """s = alpha r_c = 6.5: pair distances reach past the erfcx table's end
    (x < 6), so the pair kernel keeps the libdevice arm (the branch-free form is
    only taken when alpha r_c < 6); 15 x 15 runs the cell list, 11 x 11 the
    all-pairs kernel."""
    rng = np.random.default_rng(11)
    box = pk.BoxGeometry(box_xy, box_xy, 6.0)
    n = 700
    s = pk.make_system(np.where(np.arange(n) % 2 == 0, 1.0, -1.0), np.ones(n),
                       rng.uniform([0, 0, 0.2], [box_xy, box_xy, 5.8], size=(n, 3)), box)
    alpha = 1.6
    params = pk.make_ewald_params(alpha, 6.5, box)
    assert params.alpha * params.r_c >= 6.0
    soe = pk.build_soe_contour(8)
    modes = pk.ModeSampler(alpha, box, seed=3).batch(5)
    H = pk.normalization_H(alpha, box)
    bd, f = pk.rb_energy_forces(s, box, params, soe, _Stub(modes), 5, H=H, c_q=0.0)
    e_ref, f_ref = _oracle_eval(pk, s, box, params, soe, modes,
                                (H / 5) * (2 / np.sqrt(np.pi)) * alpha, 0.0)
    _check(bd, f, e_ref, f_ref)


@pytest.fixture(scope="module")
def big(pk):
    from paper_2403_01521_b200.configs import make_workload
    return make_workload("cfg5_1e7")


def _eval(pk, wl, s, modes):
    params = wl.params()
    soe = pk.build_soe_contour(wl.m)
    H = pk.normalization_H(wl.alpha, wl.box)
    return pk.rb_energy_forces(s, wl.box, params, soe, _Stub(modes), wl.P, H=H, c_q=0.0)


def test_size_independent_identities_at_1e7(pk, big):
    """N = 1e7 (cfg5): charge scaling by lambda scales every energy term and the
    forces by lambda^2 exactly up to rounding; a uniform in-plane translation
    (periodic) leaves energies and forces unchanged; the total force of a
    neutral slab without wall charges vanishes (Newton's third law, all terms)."""
    wl = big
    modes = pk.ModeSampler(wl.alpha, wl.box, seed=wl.seed).batch(wl.P)
    bd, f = _eval(pk, wl, wl.system, modes)
    fmax = np.max(np.abs(f))
    lam = 1.5
    s2 = pk.make_system(wl.system.charge * lam, wl.system.mass, wl.system.pos, wl.box)
    bd2, f2 = _eval(pk, wl, s2, modes)
    for k in ("u_s", "u_l_k", "u_l_0", "u_self", "u_ps"):
        a, b = getattr(bd, k) * lam ** 2, getattr(bd2, k)
        assert abs(a - b) <= 1e-11 * max(abs(a), 1.0), k
    assert np.max(np.abs(f * lam ** 2 - f2)) <= 1e-11 * lam ** 2 * fmax
    shift = np.array([0.37 * wl.box.lx, 0.61 * wl.box.ly, 0.0])
    s3 = pk.make_system(wl.system.charge, wl.system.mass, wl.system.pos + shift, wl.box)
    bd3, f3 = _eval(pk, wl, s3, modes)
    assert abs(bd3.total - bd.total) <= 1e-10 * abs(bd.total)
    assert np.max(np.abs(f3 - f)) <= 1e-9 * fmax
    assert np.all(np.abs(f.sum(axis=0)) <= 1e-9 * fmax * np.sqrt(wl.n))


@pytest.mark.parametrize("n", [3000, 40000])
def test_unwrapped_and_edge_positions_short_range(pk, n):
    """Short range on positions outside the primary cell (a system built without
    a box, MD floor-wrap leftovers) and exactly on the upper box edge: the
    reference's minimum image makes u_s and the forces independent of the
    periodic image each particle is given in (such particles used
    to be filed in a cell their fp32 screen copy did not lie in)."""
    rng = np.random.default_rng(n)
    box = pk.BoxGeometry(*(3 * [(n / 0.1) ** (1.0 / 3.0)]))
    pos = rng.random((n, 3)) * np.array([box.lx, box.ly, box.lz])
    q = np.where(np.arange(n) % 2 == 0, 1.0, -1.0)
    alpha, rc = 0.8, 4.0
    pos[:5, 0] = box.lx * (1 - 1e-16 * np.arange(5))   # on / just below the upper x edge
    pos[5:10, 1] = np.nextafter(box.ly, 0.0)            # just below the upper y edge
    base = pk.make_system(q, np.ones(n), pos, box)
    u0, f0 = pk.short_range_energy_forces(base, box, alpha, rc)
    img = pos.copy()
    k = rng.integers(-2, 3, size=(n, 2)).astype(np.float64)
    img[:, 0] += k[:, 0] * box.lx                       # other periodic images, unwrapped
    img[:, 1] += k[:, 1] * box.ly
    shifted = pk.ParticleSystem(q, np.ones(n), img, np.zeros((n, 3)))   # no wrap
    u1, f1 = pk.short_range_energy_forces(shifted, box, alpha, rc)
    assert abs(u1 - u0) <= 1e-11 * abs(u0)
    assert np.max(np.abs(f1 - f0)) <= 1e-10 * np.max(np.abs(f0))


@pytest.mark.parametrize("squeeze", [0.2, 0.6])
def test_neighbour_overflow_mid_run_matches_oracle(pk, squeeze):
    """A device-resident evaluator whose capacity was learned on a uniform slab,
    then fed a compressed one (local density x 1/squeeze, rows overflow) with no
    warm-up or rerun: the overflowed homes are evaluated in-stream
    (overflow_pairs_kernel), so energies and forces still match the oracle and
    the status only reports the overflow (verdict r01, weak 6 / next 7)."""
    import torch
    from paper_2403_01521_b200 import _native
    from paper_2403_01521_b200.configs import make_workload
    from paper_2403_01521_b200.engine import DeviceEvaluator
    from paper_2403_01521_b200.rbse2d import _rb_commonv
    wl = make_workload("cfg5_1e4")
    soe = pk.build_soe_contour(wl.m)
    params = wl.params()
    modes = pk.ModeSampler(wl.alpha, wl.box, seed=9).batch(wl.P)
    H = pk.normalization_H(wl.alpha, wl.box)
    cq = 1.25
    ev = DeviceEvaluator(wl.system, wl.box, params, soe, P=wl.P, H=H, c_q=cq, modes=modes,
                         sample=False)
    ev.warmup()
    pos2 = wl.system.pos.copy()
    z0 = 0.5 * wl.box.lz * (1.0 - squeeze)
    pos2[:, 2] = z0 + squeeze * pos2[:, 2]   # squeeze every height towards the middle
    ev.set_positions(torch.as_tensor(pos2))
    e, f = ev.step()
    torch.cuda.synchronize()
    st = ev.status()
    assert st & _native.SLAB_STATUS_NBR_OVERFLOW, "the squeeze was meant to overflow rows"
    s2 = pk.make_system(wl.system.charge, wl.system.mass, pos2, wl.box)
    e_ref, f_ref = _oracle_eval(pk, s2, wl.box, params, soe, modes,
                                _rb_commonv(H, wl.P, wl.alpha), cq)
    e = e.cpu().numpy()
    bd = pk.EnergyBreakdown(*[float(x) for x in e[:5]])
    _check(bd, f.cpu().numpy(), e_ref, f_ref)


def test_lone_complex_soe_table_matches_reference(pk):
    """soe_energy_forces with lone complex SOE terms against the REAL reference's
    output (tests/golden/lone_soe.npz)."""
    from helpers import load_golden
    g = load_golden("lone_soe")
    box = pk.BoxGeometry(*[float(v) for v in g["box"]])
    s = pk.make_system(g["q"], np.ones(len(g["q"])), g["pos"], box)
    params = pk.make_ewald_params(float(g["alpha"]), float(g["s_par"]), box)
    soe = pk.SOEApprox(m=3, w=g["w"], s=g["s"], eps_certified=1.0, domain_max=20.0)
    bd, f = pk.soe_energy_forces(s, box, params, soe)
    _check(bd, f, [float(g[k]) for k in ("u_s", "u_l_k", "u_l_0", "u_self", "u_ps")],
           g["forces"])
