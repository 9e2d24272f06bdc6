"""GPU: the device-resident MD step against the REAL
reference's md.py outputs (tests/golden/md.npz, made by make_golden.py md):
WCA core on both pair paths, walls, and short deterministic trajectories
(thermostat none / Nose-Hoover, Coulomb by soewald2d); plus the Langevin
kernel against the numpy step and its thermostat statistics."""

import numpy as np
import pytest

from helpers import load_golden

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def pk():
    import paper_2403_01521_b200 as pk
    return pk


@pytest.fixture(scope="module")
def g():
    return load_golden("md")


def test_wca_matches_reference_brute_and_cells(pk, g):
    from paper_2403_01521_b200 import md
    for tag, box, eps, sig in (("b", pk.BoxGeometry(2.0, 2.0, 3.0), 1.0, 1.0),
                               ("c", pk.BoxGeometry(12.0, 12.0, 6.0), 1.3, 0.9)):
        pos = g[f"wca_{tag}_pos"]
        s = pk.make_system(np.ones(len(pos)), np.ones(len(pos)), pos)
        u, f = md.lj_forces(s, box, eps, sig)
        assert u == pytest.approx(float(g[f"wca_{tag}_u"]), rel=1e-12)
        ref = g[f"wca_{tag}_f"]
        np.testing.assert_allclose(f, ref, rtol=0, atol=1e-12 * np.max(np.abs(ref)))


def test_walls_match_reference_and_errors(pk, g):
    from paper_2403_01521_b200 import md
    box = pk.BoxGeometry(12.0, 12.0, 6.0)
    pos = g["walls_pos"]
    s = pk.make_system(np.ones(len(pos)), np.ones(len(pos)), pos)
    u, f = md.wall_forces(s, box, 1.0, 0.5)
    assert u == pytest.approx(float(g["walls_u"]), rel=1e-12)
    np.testing.assert_allclose(f, g["walls_f"], rtol=0, atol=1e-12 * np.max(np.abs(g["walls_f"])))
    bad = pos.copy()
    bad[3, 2] = 0.0
    with pytest.raises(ValueError, match="beyond a wall"):
        md.wall_forces(pk.make_system(np.ones(len(pos)), np.ones(len(pos)), bad), box)
    two = np.array([[1.0, 1.0, 2.0], [1.0, 1.0, 2.0]])
    with pytest.raises(ValueError, match="repulsive core"):
        md.lj_forces(pk.make_system(np.ones(2), np.ones(2), two), pk.BoxGeometry(2.0, 2.0, 4.0))


@pytest.mark.parametrize("thermo", ["none", "nose-hoover"])
def test_deterministic_trajectories_match_reference(pk, g, thermo):
    """20 velocity-Verlet (or Nose-Hoover) steps with Coulomb (soewald2d) + WCA +
    walls, no random numbers: the whole trajectory follows the reference."""
    from paper_2403_01521_b200 import md
    box = pk.BoxGeometry(8.0, 8.0, 6.0)
    charge = np.array([1.0, -1.0] * 32)
    s = pk.ParticleSystem(charge=charge, mass=np.ones(64), pos=g["traj_pos0"].copy(),
                          vel=g["traj_vel0"].copy())
    opts = md.MDOptions(dt=0.002, n_steps=20, thermostat=thermo, solver="soewald2d", alpha=1.0,
                        s=3.0, soe_size=8, sample_every=5, seed=3)
    res = md.run_simulation(s, box, opts)
    key = thermo.replace("-", "")
    np.testing.assert_allclose(res.positions, g[f"traj_{key}_pos"], rtol=0, atol=1e-10)
    np.testing.assert_allclose(res.unwrapped, g[f"traj_{key}_unwrapped"], rtol=0, atol=1e-10)
    np.testing.assert_allclose(res.velocities, g[f"traj_{key}_vel"], rtol=0, atol=1e-9)
    np.testing.assert_allclose(res.potential, g[f"traj_{key}_pot"], rtol=1e-10)
    np.testing.assert_allclose(res.kinetic, g[f"traj_{key}_kin"], rtol=1e-10)
    np.testing.assert_allclose(res.conserved, g[f"traj_{key}_cons"], rtol=1e-10)
    obs = md.compute_observables(res, n_bins=8, n_blocks=2)
    assert obs["msd_xy"].shape == obs["msd_z"].shape and np.all(obs["msd_xy"] >= 0)


def test_langevin_kernel_is_the_numpy_step_without_noise(pk):
    """gamma = 0: c = 1 and no noise -- the device step equals md.langevin_step."""
    import torch
    from paper_2403_01521_b200 import md
    from paper_2403_01521_b200.engine import get_engine
    rng = np.random.default_rng(2)
    n = 500
    box = pk.BoxGeometry(10.0, 10.0, 5.0)
    pos = rng.uniform([0, 0, 1], [10, 10, 4], size=(n, 3))
    vel = rng.normal(size=(n, 3))
    frc = rng.normal(size=(n, 3))
    mass = rng.uniform(0.5, 2.0, n)
    want_p, want_v = md.langevin_step(pos, vel, frc, mass, 0.01, 0.0, 1.0, np.zeros((n, 3)))
    want_p[:, 0] -= np.floor(want_p[:, 0] / box.lx) * box.lx
    want_p[:, 1] -= np.floor(want_p[:, 1] / box.ly) * box.ly
    eng = get_engine()
    d = lambda a: torch.tensor(a, dtype=torch.float64, device=eng.device)
    P, V, F, M = d(pos), d(vel), d(frc), d(mass)
    ctr = torch.zeros(1, dtype=torch.int64, device=eng.device)
    sh = torch.zeros((n, 2), dtype=torch.float64, device=eng.device)
    eng.md_langevin(P, V, F, M, 0.01, 0.0, 1.0, 7, ctr, sh, box)
    np.testing.assert_allclose(P.cpu().numpy(), want_p, rtol=0, atol=1e-14)
    np.testing.assert_allclose(V.cpu().numpy(), want_v, rtol=0, atol=1e-14)
    assert int(ctr.item()) == 1


def test_langevin_thermalises_free_particles(pk):
    """No interactions: the OU stage alone must bring <K> to 3/2 N T, and the
    noise stream must be reproducible per seed."""
    from paper_2403_01521_b200 import md
    rng = np.random.default_rng(4)
    n = 4000
    box = pk.BoxGeometry(50.0, 50.0, 20.0)
    pos = rng.uniform([0, 0, 8], [50, 50, 12], size=(n, 3))  # far from the walls
    s = pk.ParticleSystem(charge=np.zeros(n), mass=np.full(n, 2.0), pos=pos,
                          vel=np.full((n, 3), 1e-3))
    opts = md.MDOptions(dt=0.01, n_steps=400, thermostat="langevin", gamma=5.0,
                        temperature=1.7, coulomb=False, lj_eps=0.0, wall_eps=0.0,
                        sample_every=100, seed=9)
    r1 = md.run_simulation(s, box, opts)
    r2 = md.run_simulation(s, box, opts)
    np.testing.assert_array_equal(r1.velocities, r2.velocities)
    kin = r1.kinetic[-1]
    assert kin == pytest.approx(1.5 * n * 1.7, rel=0.05)
    assert np.all(np.isnan(r1.conserved))


def test_rbse2d_langevin_run_is_finite(pk):
    from paper_2403_01521_b200 import md
    rng = np.random.default_rng(6)
    n = 200
    box = pk.BoxGeometry(14.0, 14.0, 8.0)
    g3 = np.stack(np.meshgrid(np.arange(10) * 1.4 + 0.5, np.arange(10) * 1.4 + 0.5,
                              [2.5, 5.5], indexing="ij"), -1).reshape(-1, 3)
    s = pk.make_system(np.array([1.0, -1.0] * 100), np.ones(n),
                       g3 + rng.uniform(-0.1, 0.1, g3.shape), box=box)
    opts = md.MDOptions(dt=0.002, n_steps=30, thermostat="langevin", solver="rbse2d",
                        alpha=1.0, s=3.0, batch_size=16, sample_every=10, seed=1)
    res = md.run_simulation(s, box, opts)
    assert np.all(np.isfinite(res.potential)) and np.all(np.isfinite(res.positions))
    assert np.all((res.positions[..., 2] > 0) & (res.positions[..., 2] < box.lz))


def test_ewald2d_solver_trajectory_matches_reference(pk):
    """MD with solver="ewald2d" (reference md.py:149-150): the device O(N^2 K)
    Ewald2D force field enqueued in the device-resident loop follows the
    reference's 20-step NVE trajectory (tests/golden/md_ewald.npz)."""
    from paper_2403_01521_b200 import md
    g = load_golden("md_ewald")
    box = pk.BoxGeometry(8.0, 8.0, 6.0)
    charge = np.array([1.0, -1.0] * 32)
    s = pk.ParticleSystem(charge=charge, mass=np.ones(64), pos=g["pos0"].copy(),
                          vel=g["vel0"].copy())
    opts = md.MDOptions(dt=0.002, n_steps=20, thermostat="none", solver="ewald2d", alpha=1.0,
                        s=3.0, sample_every=5, seed=3)
    res = md.run_simulation(s, box, opts)
    np.testing.assert_allclose(res.positions, g["pos"], rtol=0, atol=1e-10)
    np.testing.assert_allclose(res.velocities, g["vel"], rtol=0, atol=1e-9)
    np.testing.assert_allclose(res.potential, g["pot"], rtol=1e-10)
    np.testing.assert_allclose(res.kinetic, g["kin"], rtol=1e-10)
    np.testing.assert_allclose(res.conserved, g["cons"], rtol=1e-10)
