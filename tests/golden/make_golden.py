"""Generate golden fixtures by running the REAL reference package (in the build container).

The reference (``/root/reference/pkg/src/slabewald``) is pure Python + numba and
cannot travel to the GPU box, so its outputs on our seeded workloads are frozen
here as small ``.npz`` fixtures.  Usage (build container only)::

    NUMBA_CACHE_DIR=/tmp/numba_cache python tests/golden/make_golden.py [names...]

Inputs are regenerated from ``paper_2403_01521_b200.configs.make_workload`` (a
sha256 of positions/charges is stored so a test can prove the regeneration is
bit-identical).  Random-batch k-sets are drawn ONCE from the reference
``ModeSampler`` and injected into ``rb_energy_forces`` through a stub whose
``batch(P)`` returns them (``rbse2d.py:288`` only calls ``sampler.batch(P)``).
"""

from __future__ import annotations

import hashlib
import importlib.util
import os
import sys
import time

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
REPO = os.path.dirname(os.path.dirname(HERE))
REF_SRC = "/root/reference/pkg/src"

FULL_LIMIT = 20_000       # store full force / perm arrays up to this N
N_SAMPLE = 4096           # otherwise a fixed random subset of particles


def _load_pkg_module(name):
    """Import one host module of our package without triggering its __init__
    (which loads the CUDA library)."""
    pkg = "paper_2403_01521_b200"
    if pkg not in sys.modules:
        spec = importlib.util.spec_from_file_location(
            pkg, os.path.join(REPO, pkg, "__init__.py"),
            submodule_search_locations=[os.path.join(REPO, pkg)])
        mod = importlib.util.module_from_spec(spec)
        sys.modules[pkg] = mod  # bare namespace, __init__ not executed
    full = f"{pkg}.{name}"
    spec = importlib.util.spec_from_file_location(full, os.path.join(REPO, pkg, f"{name}.py"))
    mod = importlib.util.module_from_spec(spec)
    sys.modules[full] = mod
    spec.loader.exec_module(mod)
    return mod


def sha(a: np.ndarray) -> str:
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


class StubSampler:
    def __init__(self, modes):
        self.modes = modes

    def batch(self, P):
        assert P == self.modes.shape[0]
        return self.modes


def ref_modules():
    os.environ.setdefault("NUMBA_CACHE_DIR", "/tmp/numba_cache")
    if REF_SRC not in sys.path:
        sys.path.insert(0, REF_SRC)
    import slabewald  # noqa: F401
    from slabewald import core, ewald2d, rbse2d, soe, soewald2d
    return core, ewald2d, rbse2d, soe, soewald2d


def golden_workload(name: str) -> dict:
    core, ewald2d, rbse2d, rsoe, soewald2d = ref_modules()
    configs = _load_pkg_module("core") and _load_pkg_module("configs")
    wl = configs.make_workload(name)
    b = wl.box
    box = core.BoxGeometry(b.lx, b.ly, b.lz, b.sigma_top, b.sigma_bot)
    sysm = core.make_system(wl.system.charge, wl.system.mass, wl.system.pos, box=box)
    assert np.array_equal(sysm.pos, wl.system.pos)
    params = core.make_ewald_params(wl.alpha, wl.s, box)
    soe = rsoe.build_soe_contour(wl.m)
    out = dict(name=name, n=wl.n, alpha=wl.alpha, s=wl.s, m=wl.m,
               box=np.array([b.lx, b.ly, b.lz, b.sigma_top, b.sigma_bot]),
               pos_sha=sha(wl.system.pos), charge_sha=sha(wl.system.charge),
               soe_w=soe.w, soe_s=soe.s)
    t0 = time.perf_counter()
    if wl.P is None:
        bd, forces = soewald2d.soe_energy_forces(sysm, box, params, soe)
        out["modes"] = params.kmodes
        out["P"] = 0
    else:
        sampler = rbse2d.ModeSampler(wl.alpha, box, seed=wl.seed)
        modes = sampler.batch(wl.P)
        H = rbse2d.normalization_H(wl.alpha, box)
        c_q = rbse2d.charge_term_sum(wl.alpha, box, float(np.sum(sysm.charge ** 2)))
        bd, forces = rbse2d.rb_energy_forces(sysm, box, params, soe, StubSampler(modes),
                                             wl.P, H=H, c_q=c_q)
        out.update(modes=modes, P=wl.P, H=H, c_q=c_q)
    out["seconds"] = time.perf_counter() - t0
    u_s, f_s = ewald2d.short_range_energy_forces(sysm, box, wl.alpha, params.r_c)
    perm = core.sort_by_z(sysm, box.lz)
    for k in ("u_s", "u_l_k", "u_l_0", "u_self", "u_ps"):
        out[k] = getattr(bd, k)
    out["total"] = bd.total
    out["u_s_alone"] = u_s
    out["fmax"] = float(np.max(np.abs(forces)))
    out["fsum"] = forces.sum(axis=0)
    out["fabs"] = np.abs(forces).sum(axis=0)
    out["perm_sha"] = sha(perm.astype(np.int64))
    if wl.n <= FULL_LIMIT:
        out["forces"] = forces
        out["f_short"] = f_s
        out["perm"] = perm.astype(np.int64)
    else:
        idx = np.sort(np.random.default_rng(12345).choice(wl.n, N_SAMPLE, replace=False))
        out["sample_idx"] = idx
        out["forces"] = forces[idx]
        out["f_short"] = f_s[idx]
        out["perm_head"] = perm[:N_SAMPLE].astype(np.int64)
    return out


def golden_units() -> dict:
    """Small known-answer vectors: sort edge cases, recursion, sampler, H / C_Q."""
    core, ewald2d, rbse2d, rsoe, soewald2d = ref_modules()
    out = {}
    rng = np.random.default_rng(2024)
    cases = {
        "sort_small": np.array([3.0, 1.0, 2.0]),
        "sort_ties": np.array([1.0, 0.25, 1.0, 0.25, 1.0]),
        "sort_negzero": np.array([0.0, -0.0, 0.5, -0.0, 0.0, 2.0, 2.0]),
        "sort_random": rng.random(10_000) * 6.0,
        "sort_clustered": np.round(rng.random(5000) * 7.0, 2),
        "sort_reversed": np.linspace(5.0, 0.0, 3001),
        "sort_top": np.array([4.0, 0.0, 4.0, 2.0, 4.0]),
    }
    for k, z in cases.items():
        n = len(z)
        lz = float(max(z.max(), 1.0))
        pos = np.column_stack([np.zeros(n), np.zeros(n), z])
        sysm = core.make_system(np.ones(n), np.ones(n), pos)
        out[k + "_z"] = z
        out[k + "_lz"] = lz
        out[k + "_perm"] = core.sort_by_z(sysm, lz).astype(np.int64)
    # recursive_pair_sum known answers
    n = 64
    q = rng.choice([-1.0, 1.0], size=n)
    th = rng.uniform(-np.pi, np.pi, size=n)
    z = np.sort(rng.uniform(0.0, 8.0, size=n))
    for j, beta in enumerate([0.3 + 0.7j, 1.1 + 0.0j, 0.05 - 2.0j]):
        out[f"rps_{j}_beta"] = np.array(beta)
        out[f"rps_{j}_out"] = soewald2d.recursive_pair_sum(q, th, z, beta)
    out["rps_q"], out["rps_theta"], out["rps_z"] = q, th, z
    # H, C_Q over a spread of boxes
    hv = []
    for a, lx, ly in [(0.3, 100.0, 100.0), (0.464, 58.48, 58.48), (0.8, 10.0, 13.0),
                      (0.05, 100.0, 100.0), (0.5, 20.0, 20.0)]:
        box = core.BoxGeometry(lx, ly, 10.0)
        import warnings
        with warnings.catch_warnings():
            warnings.simplefilter("ignore")
            hv.append([a, lx, ly, rbse2d.normalization_H(a, box),
                       rbse2d.charge_term_sum(a, box, 50.0)])
    out["H_cq_table"] = np.array(hv)
    # reference sampler draws (statistical comparison only: different RNG stream)
    box = core.BoxGeometry(100.0, 100.0, 10.0)
    smp = rbse2d.ModeSampler(0.3, box, seed=11)
    out["sampler_idx_a03_L100_seed11"] = smp.batch_indices(20000)
    out["sampler_acc_a03_L100_seed11"] = smp.acceptance_rate
    # single-mode energies on a small slab (fourier_mode_energy_soe, soe8)
    box = core.BoxGeometry(20.0, 20.0, 10.0)
    rng2 = np.random.default_rng(21)
    posm = rng2.uniform([0.0, 0.0, 0.5], [20.0, 20.0, 9.5], size=(20, 3))
    qm = np.array([1.0, -1.0] * 10)
    sysm = core.make_system(qm, np.ones(20), posm, box=box)
    params = core.make_ewald_params(0.5, 3.0, box)
    soe8 = rsoe.build_soe_contour(8)
    out["mode_pos"], out["mode_q"] = posm, qm
    out["mode_energies"] = np.array([soewald2d.fourier_mode_energy_soe(sysm, box, params, soe8, i)
                                     for i in range(params.kmodes.shape[0])])
    out["mode_zero"] = soewald2d.zero_mode_energy_soe(sysm, box, 0.5, soe8)
    bd, f = soewald2d.soe_energy_forces(sysm, box, params, soe8)
    out["mode_total"] = bd.total
    out["mode_forces"] = f
    out["mode_forces_soe"] = soewald2d.forces_soe(sysm, box, params, soe8)
    return out


def md_system(seed=11):
    """64 charges +-1 on a jittered 4x4x4 lattice in (8, 8, 6), seeded velocities."""
    rng = np.random.default_rng(seed)
    g = (np.arange(4) + 0.5)
    lat = np.stack(np.meshgrid(g * 2.0, g * 2.0, g * 1.5 - 0.0, indexing="ij"), -1).reshape(-1, 3)
    pos = lat + rng.uniform(-0.25, 0.25, size=lat.shape)
    charge = np.array([1.0, -1.0] * 32)
    vel = rng.normal(size=(64, 3)) * 0.7
    return charge, np.ones(64), pos, vel


def golden_md() -> dict:
    """md.py: WCA core (brute and cell paths), walls, and short deterministic
    trajectories (thermostat none / nose-hoover: no random numbers)."""
    core, ewald2d, rbse2d, rsoe, soewald2d = ref_modules()
    from slabewald import md
    out = {}
    rng = np.random.default_rng(5)
    # WCA, brute path (reference: ncx == 1 when L < 2 cut)
    box_b = core.BoxGeometry(2.0, 2.0, 3.0)
    pos_b = rng.uniform([0, 0, 0.3], [2.0, 2.0, 2.7], size=(10, 3))
    sb = core.make_system(np.ones(10), np.ones(10), pos_b, box=box_b)
    out["wca_b_pos"] = sb.pos
    out["wca_b_u"], out["wca_b_f"] = md.lj_forces(sb, box_b, 1.0, 1.0)
    # WCA, cell path
    box_c = core.BoxGeometry(12.0, 12.0, 6.0)
    pos_c = rng.uniform([0, 0, 0.2], [12.0, 12.0, 5.8], size=(300, 3))
    sc = core.make_system(np.ones(300), np.ones(300), pos_c, box=box_c)
    out["wca_c_pos"] = sc.pos
    out["wca_c_u"], out["wca_c_f"] = md.lj_forces(sc, box_c, 1.3, 0.9)
    # walls
    zw = np.concatenate([rng.uniform(0.05, 0.6, 20), rng.uniform(5.4, 5.95, 20),
                         rng.uniform(1.0, 5.0, 20)])
    pos_w = np.column_stack([rng.uniform(0, 12, 60), rng.uniform(0, 12, 60), zw])
    sw = core.make_system(np.ones(60), np.ones(60), pos_w, box=box_c)
    out["walls_pos"] = sw.pos
    out["walls_u"], out["walls_f"] = md.wall_forces(sw, box_c, 1.0, 0.5)
    # deterministic trajectories
    charge, mass, pos, vel = md_system()
    box = core.BoxGeometry(8.0, 8.0, 6.0)
    out["traj_pos0"], out["traj_vel0"] = pos, vel
    for thermo in ("none", "nose-hoover"):
        sysm = core.ParticleSystem(charge=charge, mass=mass, pos=pos.copy(), vel=vel.copy())
        opts = md.MDOptions(dt=0.002, n_steps=20, thermostat=thermo, solver="soewald2d",
                            alpha=1.0, s=3.0, soe_size=8, sample_every=5, seed=3)
        res = md.run_simulation(sysm, box, opts)
        key = thermo.replace("-", "")
        out[f"traj_{key}_pos"] = res.positions
        out[f"traj_{key}_unwrapped"] = res.unwrapped
        out[f"traj_{key}_vel"] = res.velocities
        out[f"traj_{key}_pot"] = res.potential
        out[f"traj_{key}_kin"] = res.kinetic
        out[f"traj_{key}_cons"] = res.conserved
    return out


def golden_md_ewald() -> dict:
    """md.py with solver="ewald2d" (md.py:149-150, the O(N^2 K) reference solver as
    the force field): a 20-step NVE trajectory of the md_system slab."""
    core, ewald2d, rbse2d, rsoe, soewald2d = ref_modules()
    from slabewald import md
    charge, mass, pos, vel = md_system()
    box = core.BoxGeometry(8.0, 8.0, 6.0)
    sysm = core.ParticleSystem(charge=charge, mass=mass, pos=pos.copy(), vel=vel.copy())
    opts = md.MDOptions(dt=0.002, n_steps=20, thermostat="none", solver="ewald2d", alpha=1.0,
                        s=3.0, sample_every=5, seed=3)
    res = md.run_simulation(sysm, box, opts)
    return dict(pos0=pos, vel0=vel, pos=res.positions, unwrapped=res.unwrapped,
                vel=res.velocities, pot=res.potential, kin=res.kinetic, cons=res.conserved)


def golden_lone_soe() -> dict:
    """soe_energy_forces (soewald2d.py:398-438) with an SOE table whose complex
    terms have no conjugate partners -- the reference sweep takes any (w, s)."""
    core, ewald2d, rbse2d, rsoe, soewald2d = ref_modules()
    rng = np.random.default_rng(31)
    box = core.BoxGeometry(15.0, 15.0, 6.0)
    n = 300
    pos = rng.uniform([0, 0, 0.2], [15, 15, 5.8], size=(n, 3))
    q = np.where(np.arange(n) % 2 == 0, 1.0, -1.0)
    sysm = core.make_system(q, np.ones(n), pos, box=box)
    w = np.array([0.7 - 0.2j, 0.3 + 0.9j, 1.1 + 0.1j])
    sv = np.array([1.5 + 0.8j, 2.5 - 1.7j, 0.9 + 3.0j])
    soe = rsoe.SOEApprox(m=3, w=w, s=sv, eps_certified=1.0, domain_max=20.0)
    params = core.make_ewald_params(0.9, 3.0, box)
    bd, f = soewald2d.soe_energy_forces(sysm, box, params, soe)
    return dict(pos=sysm.pos, q=q, w=w, s=sv, alpha=0.9, s_par=3.0, box=np.array([15.0, 15.0, 6.0]),
                u_s=bd.u_s, u_l_k=bd.u_l_k, u_l_0=bd.u_l_0, u_self=bd.u_self, u_ps=bd.u_ps,
                forces=f)


def golden_ewald_ref() -> dict:
    """ewald2d.py: the O(N^2 K) Ewald2D reference on two small neutral systems
    (stable and naive xi kernels, k = 0 mode, full breakdown)."""
    core, ewald2d, rbse2d, rsoe, soewald2d = ref_modules()
    out = {}
    for tag, n, box_l, alpha, s_par, seed in (("a", 60, (10.0, 10.0, 5.0), 0.6, 3.0, 21),
                                              ("b", 200, (14.0, 11.0, 7.0), 0.8, 3.5, 22)):
        rng = np.random.default_rng(seed)
        box = core.BoxGeometry(*box_l)
        pos = rng.uniform([0, 0, 0.2], [box_l[0], box_l[1], box_l[2] - 0.2], size=(n, 3))
        q = np.where(np.arange(n) % 2 == 0, 1.0, -1.0)
        sysm = core.make_system(q, np.ones(n), pos, box=box)
        params = core.make_ewald_params(alpha, s_par, box)
        bd, f = ewald2d.ref_energy_forces(sysm, box, params)
        out[f"{tag}_pos"] = sysm.pos
        out[f"{tag}_nmode"] = params.kmodes.shape[0]
        for k in ("u_s", "u_l_k", "u_l_0", "u_self", "u_ps"):
            out[f"{tag}_{k}"] = getattr(bd, k)
        out[f"{tag}_forces"] = f
        uk, fk = ewald2d.fourier_energy_forces_ref(sysm, box, params, "naive")
        out[f"{tag}_naive_u"], out[f"{tag}_naive_f"] = uk, fk
        u0, f0 = ewald2d.zero_mode_energy_forces_ref(sysm, box, alpha)
        out[f"{tag}_zero_u"], out[f"{tag}_zero_f"] = u0, f0
    return out


def golden_batches() -> dict:
    """rbse2d.py:320-363 run_many_batches, with the k-sequence drawn once from the
    reference sampler and injected: per-batch forward-sweep energies from the
    reference's own _rb_batch_energy_kernel, plus u_det.  N = 1e4, P = 100 and
    41 batches: one full device pass of 40 batches and a 1-batch tail pass (the
    plan-mismatch case of ADVICE r01)."""
    core, ewald2d, rbse2d, rsoe, soewald2d = ref_modules()
    configs = _load_pkg_module("core") and _load_pkg_module("configs")
    wl = configs.make_workload("cfg5_1e4")
    b = wl.box
    box = core.BoxGeometry(b.lx, b.ly, b.lz, b.sigma_top, b.sigma_bot)
    sysm = core.make_system(wl.system.charge, wl.system.mass, wl.system.pos, box=box)
    params = core.make_ewald_params(wl.alpha, wl.s, box)
    soe = rsoe.build_soe_contour(wl.m)
    P, nb = 100, 41
    alpha = params.alpha
    H = rbse2d.normalization_H(alpha, box)
    Q = float(np.sum(sysm.charge ** 2))
    c_q = rbse2d.charge_term_sum(alpha, box, Q)
    u_s, _ = ewald2d.short_range_energy_forces(sysm, box, alpha, params.r_c)
    u_ps, _ = ewald2d.slab_energy_forces(sysm, box)
    u_det = (u_s + soewald2d.zero_mode_energy_soe(sysm, box, alpha, soe)
             - ewald2d.self_energy(sysm, alpha) + u_ps + c_q)
    sampler = rbse2d.ModeSampler(alpha, box, seed=31)
    rec = sampler.batch_indices(nb * P)
    kx = 2 * np.pi * rec[:, 0] / box.lx
    ky = 2 * np.pi * rec[:, 1] / box.ly
    kv = np.hypot(kx, ky)
    _, x, yv, z, q = soewald2d._sorted_view(sysm, box)
    bvec = alpha * soe.s
    decays = soewald2d._decay_table(z, bvec)
    commonv = np.full(nb * P, (H / P) * rbse2d.TWO_OVER_SQRT_PI * alpha)
    out = np.empty(nb)
    rbse2d._rb_batch_energy_kernel(x, yv, z, q, kx, ky, kv, commonv, soe.w, bvec, box.area,
                                   decays, P, out)
    return dict(n=wl.n, P=P, n_batches=nb, H=H, c_q=c_q, u_det=u_det,
                modes=np.column_stack([kx, ky, kv]), batch_u=out,
                estimates=out + u_det, pos_sha=sha(wl.system.pos))


def golden_formats() -> dict:
    """Files WRITTEN by the reference (core.py:305-329 save_particles, soe.py:172-177
    save_soe_table), their text and the reference's own load of them, for
    cross-checking this package's readers and writers."""
    import tempfile
    core, ewald2d, rbse2d, rsoe, soewald2d = ref_modules()
    rng = np.random.default_rng(77)
    n = 37
    pos = rng.uniform(-3.0, 13.0, size=(n, 3))
    pos[:, 2] = rng.uniform(0.0, 6.0, size=n)
    pos[0] = [0.0, -0.0, 6.0]
    pos[1, 0] = 1e-300
    vel = rng.normal(size=(n, 3)) * 1e3
    q = rng.choice([-2.0, 1.0, 0.5], size=n)
    m = rng.uniform(0.1, 40.0, size=n)
    box = core.BoxGeometry(10.0, 12.0, 6.0)
    sysm = core.make_system(q, m, pos, vel, box=box)
    out = {}
    with tempfile.TemporaryDirectory() as td:
        pp = os.path.join(td, "p.csv")
        core.save_particles(pp, sysm)
        out["particles_csv"] = np.array(open(pp).read())
        back = core.load_particles(pp, box=box)
        out["particles_q"], out["particles_m"] = back.charge, back.mass
        out["particles_pos"], out["particles_vel"] = back.pos, back.vel
        for mm in (8, 16):
            tp = os.path.join(td, f"s{mm}.csv")
            rsoe.save_soe_table(tp, rsoe.build_soe_contour(mm))
            out[f"soe{mm}_csv"] = np.array(open(tp).read())
            t = rsoe.load_soe_table(tp)
            out[f"soe{mm}_w"], out[f"soe{mm}_s"] = t.w, t.s
            out[f"soe{mm}_eps"] = t.eps_certified
        # a hand-made table (one real term, one complex pair) as the soe tests use
        hand = rsoe.SOEApprox(m=3, w=np.array([0.5 + 0.0j, 0.2 + 0.1j, 0.2 - 0.1j]),
                              s=np.array([1.3 + 0.0j, 0.7 + 2.0j, 0.7 - 2.0j]),
                              eps_certified=0.0, domain_max=20.0)
        hp = os.path.join(td, "hand.csv")
        rsoe.save_soe_table(hp, hand)
        out["hand_csv"] = np.array(open(hp).read())
        t = rsoe.load_soe_table(hp)
        out["hand_w"], out["hand_s"], out["hand_eps"] = t.w, t.s, t.eps_certified
    out["box"] = np.array([box.lx, box.ly, box.lz])
    out["src_pos"], out["src_vel"], out["src_q"], out["src_m"] = sysm.pos, sysm.vel, q, m
    return out


def main(argv):
    names = argv or ["units", "cfg1", "cfg2", "small_600", "small_2000", "cfg5_1e4",
                     "cfg3", "cfg5_1e5", "cfg4", "cfg5_1e6"]
    for name in names:
        t0 = time.perf_counter()
        data = (golden_units() if name == "units" else
                golden_batches() if name == "batches" else
                golden_formats() if name == "formats" else
                golden_md() if name == "md" else
                golden_md_ewald() if name == "md_ewald" else
                golden_lone_soe() if name == "lone_soe" else
                golden_ewald_ref() if name == "ewald_ref" else golden_workload(name))
        path = os.path.join(HERE, f"{name}.npz")
        np.savez_compressed(path, **{k: np.asarray(v) for k, v in data.items()})
        print(f"{name}: wrote {path} ({os.path.getsize(path)/1e3:.0f} kB) "
              f"in {time.perf_counter() - t0:.1f}s", flush=True)


if __name__ == "__main__":
    main(sys.argv[1:])
