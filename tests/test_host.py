"""CPU: host-side logic of the drop-in API (per-run setup; no device needed).

Mirrors the reference's own known-answer / relational tests for the same
functions (pkg/tests/test_core.py, test_soe.py, test_rbse2d.py) and pins the
host outputs against the reference's values frozen in tests/golden.
"""

import math
import warnings

import numpy as np
import pytest

from helpers import load_golden
import paper_2403_01521_b200 as pk
from paper_2403_01521_b200 import soe as soe_mod
from paper_2403_01521_b200.configs import make_workload
from paper_2403_01521_b200.rbse2d import _axis_logq

H_BRUTE_03_100 = 285.47889756541156   # reference tests/test_rbse2d.py:28
Q0_PROPOSAL = 0.05902784737600369     # erf(pi/60)
PROPOSAL_STD = 6.7523723711782955


def test_box_geometry_validation_and_area():
    b = pk.BoxGeometry(2.0, 3.0, 4.0)
    assert b.area == 6.0 and b.volume == 24.0
    for dims in [(0, 1, 1), (1, -1, 1), (1, 1, 0)]:
        with pytest.raises(ValueError, match="positive"):
            pk.BoxGeometry(*dims)
    with pytest.raises(ValueError, match="finite"):
        pk.BoxGeometry(1, 1, 1, sigma_top=float("nan"))


def test_make_system_wraps_xy_and_accepts_box_in_fourth_slot():
    box = pk.BoxGeometry(10.0, 10.0, 5.0)
    pos = np.array([[12.0, -3.0, 1.0], [5.0, 5.0, 5.0]])
    s1 = pk.make_system([1.0, -1.0], [1.0, 1.0], pos, box=box)
    s2 = pk.make_system([1.0, -1.0], [1.0, 1.0], pos, box)  # reference tests' call form
    np.testing.assert_array_equal(s1.pos, s2.pos)
    np.testing.assert_allclose(s1.pos[0], [2.0, 7.0, 1.0])
    with pytest.raises(ValueError, match="lie in"):
        pk.make_system([1.0], [1.0], [[1.0, 1.0, 6.0]], box)
    with pytest.raises(ValueError, match="shapes"):
        pk.make_system([1.0, 2.0], [1.0], [[1.0, 1.0, 1.0]])
    with pytest.raises(ValueError, match="positive"):
        pk.make_system([1.0], [0.0], [[1.0, 1.0, 1.0]])


def test_kmodes_match_reference_full_mode_set():
    g = load_golden("cfg1")
    wl = make_workload("cfg1")
    km = wl.params().kmodes
    assert km.shape == (792, 3)
    np.testing.assert_array_equal(km, g["modes"])
    # closed under k -> -k and excludes the origin
    s = {(round(a, 12), round(b, 12)) for a, b, _ in km}
    assert all((round(-a, 12), round(-b, 12)) in s for a, b, _ in km)
    assert not np.any(km[:, 2] == 0)


def test_ewald_params_and_alpha_laws():
    box = pk.BoxGeometry(100.0, 100.0, 100.0)
    assert pk.choose_alpha(1000, box, mode="linear") == pytest.approx(0.1, rel=1e-12)
    p = pk.make_ewald_params(0.5, 4.0, box)
    assert p.r_c == 8.0 and p.k_c == 4.0
    with pytest.raises(ValueError, match="alpha must be positive"):
        pk.make_ewald_params(0.0, 4.0, box)
    with pytest.raises(ValueError):
        pk.choose_alpha(10, box, mode="nope")


@pytest.mark.parametrize("m", [8, 16, 24])
def test_soe_contour_bitwise_equal_to_reference(m):
    g = load_golden({8: "units", 16: "cfg2", 24: "cfg3"}[m]) if m != 8 else None
    soe = pk.build_soe_contour(m)
    assert soe_mod.is_conjugate_paired(soe)
    if g is not None:
        np.testing.assert_array_equal(soe.w, g["soe_w"])
        np.testing.assert_array_equal(soe.s, g["soe_s"])
    assert soe.eps_certified <= soe_mod.ACHIEVED_EPS[m] * 1.5


def test_soe_table_roundtrip(tmp_path):
    soe = pk.build_soe_contour(8)
    path = tmp_path / "t.csv"
    pk.save_soe_table(path, soe)
    back = pk.load_soe_table(path)
    np.testing.assert_array_equal(back.w, soe.w)
    np.testing.assert_array_equal(back.s, soe.s)


def test_normalization_H_and_charge_term_match_reference_table():
    g = load_golden("units")
    for a, lx, ly, Hr, cqr in g["H_cq_table"]:
        box = pk.BoxGeometry(lx, ly, 10.0)
        with warnings.catch_warnings():
            warnings.simplefilter("ignore")
            assert pk.normalization_H(a, box) == pytest.approx(Hr, rel=1e-14)
        assert pk.charge_term_sum(a, box, 50.0) == pytest.approx(cqr, rel=1e-14)
    assert pk.normalization_H(0.3, pk.BoxGeometry(100.0, 100.0, 10.0)) == pytest.approx(
        H_BRUTE_03_100, rel=1e-9)
    with pytest.warns(UserWarning, match="Fourier modes"):
        pk.normalization_H(0.01, pk.BoxGeometry(100.0, 100.0, 10.0))
    with pytest.raises(ValueError, match="positive"):
        pk.normalization_H(0.0, pk.BoxGeometry(100.0, 100.0, 10.0))


def test_proposal_constants():
    ax = math.pi / (0.3 * 100.0)
    assert 1.0 / (ax * math.sqrt(2.0)) == pytest.approx(PROPOSAL_STD, rel=1e-12)
    assert math.exp(_axis_logq(0, ax)) == pytest.approx(Q0_PROPOSAL, rel=1e-12)
    total = sum(math.exp(_axis_logq(m, ax)) for m in range(-60, 61))
    assert total == pytest.approx(1.0, abs=1e-12)


def test_variance_diagnostics_and_csv(tmp_path):
    d = pk.variance_diagnostics(np.full(10, 2.5))
    assert d["mean"] == 2.5 and d["stderr"] == 0.0
    with pytest.raises(ValueError, match="two batches"):
        pk.variance_diagnostics(np.array([1.0]))
    est = np.random.default_rng(5).normal(size=20)
    path = tmp_path / "diag.csv"
    pk.write_diagnostics_csv(path, est)
    lines = path.read_text().strip().split("\n")
    assert lines[0] == "batch_index,estimate,running_mean,running_stderr"
    assert len(lines) == 21


def test_neutrality():
    box = pk.BoxGeometry(10.0, 10.0, 5.0)
    s = pk.make_system([1.0, -1.0], [1.0, 1.0], [[1, 1, 1], [2, 2, 2]], box)
    assert pk.validate_neutrality(s, box)[0]
    s = pk.make_system([1.0], [1.0], [[1, 1, 1]], box)
    assert not pk.validate_neutrality(s, box)[0]


def test_workload_generators_are_neutral_and_regenerate():
    for name in ("cfg1", "cfg2", "cfg3", "small_600"):
        wl = make_workload(name)
        assert abs(wl.system.charge.sum()) < 1e-9
        assert wl.system.pos[:, 2].min() >= 0 and wl.system.pos[:, 2].max() <= wl.box.lz
        wl2 = make_workload(name)
        np.testing.assert_array_equal(wl.system.pos, wl2.system.pos)


def test_particle_csv_round_trip_and_errors(tmp_path):
    """core.py:305-329 particle CSV: exact round trip, rows read back by id,
    header checked, box wrap applied on load."""
    import paper_2403_01521_b200 as pk
    rng = np.random.default_rng(3)
    pos = rng.uniform(0, 5, size=(7, 3))
    s = pk.make_system(rng.choice([-1.0, 1.0], 7), rng.uniform(1, 2, 7), pos,
                       rng.normal(size=(7, 3)))
    p = tmp_path / "p.csv"
    pk.save_particles(p, s)
    t = pk.load_particles(p)
    for a, b in ((t.pos, s.pos), (t.vel, s.vel), (t.charge, s.charge), (t.mass, s.mass)):
        np.testing.assert_array_equal(a, b)
    lines = p.read_text().splitlines()
    shuffled = tmp_path / "q.csv"
    shuffled.write_text("\n".join([lines[0]] + lines[1:][::-1]) + "\n")
    np.testing.assert_array_equal(pk.load_particles(shuffled).pos, s.pos)
    wrapped = pk.load_particles(p, box=pk.BoxGeometry(2.0, 2.0, 5.0))
    assert np.all(wrapped.pos[:, :2] < 2.0)
    bad = tmp_path / "bad.csv"
    bad.write_text("id,q,m,x,y,z\n0,1,1,0,0,0\n")
    with pytest.raises(ValueError, match="header"):
        pk.load_particles(bad)


def test_md_host_pieces_without_gpu():
    """md.py host forms: options defaults, the numpy Langevin step, observables."""
    from paper_2403_01521_b200 import md
    o = md.MDOptions()
    assert (o.dt, o.thermostat, o.solver, o.soe_size, o.batch_size) == \
        (0.005, "langevin", "soewald2d", 8, 16)
    pos = np.zeros((2, 3))
    vel = np.ones((2, 3))
    p2, v2 = md.langevin_step(pos, vel, np.zeros((2, 3)), np.ones(2), 0.1, 0.0, 1.0,
                              np.zeros((2, 3)))
    np.testing.assert_allclose(p2, 0.1 * vel)
    np.testing.assert_allclose(v2, vel)


def test_status_survives_the_sum_allreduce():
    """Slot 7 carries the status bits as 8-bit counters: summing the energy
    vectors of several ranks (the multi-GPU all-reduce) keeps every bit."""
    from paper_2403_01521_b200.ewald2d import status_of
    def vec(bits):
        v = np.zeros(8)
        v[5] = bits
        v[7] = sum(256.0 ** k for k in range(6) if bits & (1 << k))
        return v
    ranks = [vec(4), vec(4 | 1), vec(0), vec(4)]
    assert status_of(sum(ranks), summed=True) == 5
    assert status_of(vec(8)) == 8
    assert status_of(sum(vec(0) for _ in range(8)), summed=True) == 0


def test_bench_reference_arm_json_line():
    """bench.py --impl reference (the CPU arm: the C restatement on the host
    cores) runs without a GPU and prints ONE JSON line with the contract keys."""
    import json
    import os
    import subprocess
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    out = subprocess.run([sys.executable, "bench.py", "--impl", "reference", "--config", "cfg2",
                          "--steps", "1", "--warmup", "0"], cwd=root, capture_output=True,
                         text=True, timeout=600)
    assert out.returncode == 0, out.stderr[-2000:]
    lines = [ln for ln in out.stdout.splitlines() if ln.strip()]
    assert len(lines) == 1
    d = json.loads(lines[0])
    for k in ("metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step",
              "higher_is_better", "scaling", "vs_baseline", "dtype", "data", "config",
              "cpu_baseline", "e2e"):
        assert k in d, k
    assert d["impl"] == "reference" and d["value"] > 0 and d["config"]["workload"] == "cfg2"
    assert d["e2e"]["h2d_bytes_per_step"] == 0 and d["e2e"]["d2h_bytes_per_step"] == 0
    assert d["cpu_baseline"]["kind"] == "port" and d["cpu_baseline"]["cores"] >= 1


def test_formats_cross_check_with_reference_written_files(tmp_path):
    """SURVEY 8(f) rank 3 against files the REFERENCE wrote (tests/golden/formats.npz:
    core.py:305-329 save_particles, soe.py:151-177 save/load_soe_table): our
    readers load them to the reference's own arrays, our writers reproduce the
    reference's bytes, and the recertified SOE error matches."""
    from helpers import load_golden
    from paper_2403_01521_b200.core import BoxGeometry, load_particles, make_system, save_particles
    from paper_2403_01521_b200.soe import SOEApprox, load_soe_table, save_soe_table
    g = load_golden("formats")
    box = BoxGeometry(*[float(v) for v in g["box"]])
    p = tmp_path / "ref_particles.csv"
    p.write_text(str(g["particles_csv"]))
    s = load_particles(str(p), box=box)
    for ours, key in ((s.charge, "particles_q"), (s.mass, "particles_m"),
                      (s.pos, "particles_pos"), (s.vel, "particles_vel")):
        assert np.array_equal(ours, g[key]), key
    mine = tmp_path / "ours.csv"
    save_particles(str(mine), make_system(g["src_q"], g["src_m"], g["src_pos"], g["src_vel"],
                                          box=box))
    assert mine.read_text() == str(g["particles_csv"])
    for tag in ("soe8", "soe16", "hand"):
        f = tmp_path / f"{tag}.csv"
        f.write_text(str(g[f"{tag}_csv"]))
        t = load_soe_table(str(f))
        assert np.array_equal(t.w, g[f"{tag}_w"]) and np.array_equal(t.s, g[f"{tag}_s"]), tag
        assert t.eps_certified == pytest.approx(float(g[f"{tag}_eps"]), rel=1e-12), tag
        out = tmp_path / f"{tag}_ours.csv"
        save_soe_table(str(out), SOEApprox(m=len(t.w), w=t.w, s=t.s,
                                           eps_certified=t.eps_certified, domain_max=20.0))
        assert out.read_text() == str(g[f"{tag}_csv"]), tag
