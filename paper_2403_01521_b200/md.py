"""Device-resident MD engine around the evaluator.

Mirrors reference ``pkg/src/slabewald/md.py``: the same options, result record,
force field (Coulomb solver + WCA core + walls) and integrators, with the
state (positions, velocities, forces, image shifts, thermostat counter) kept on
the device between steps:

* ``lj_forces`` (md.py:34-56) -> ``slab_wca`` (short-range pair machinery with
  the WCA core, cutoff 2^(1/6) sigma);
* ``wall_forces`` (md.py:59-77) -> ``slab_walls``;
* ``langevin_step`` (md.py:180-193) -> ``slab_md_langevin`` (kick, drift, exact
  OU, drift, xy wrap with image-shift accumulation in one kernel); the final
  kick after the force evaluation -> ``slab_md_kick``;
* velocity Verlet (md.py:300-305) -> ``slab_md_kick`` / ``slab_md_drift``;
* Nose-Hoover (md.py:196-224) -> device kinetic-energy reductions and
  ``slab_md_scale``, the chain variables on the host;
* ``kinetic_energy`` (md.py:176-177) -> ``slab_md_kinetic``.

Differences, by design: the Langevin noise is a counter-based Philox4x32-10
stream keyed by the run seed (reproducible per seed, not numpy's Generator
sequence -- the policy of the mode sampler); the ``ewald2d`` solver (the O(N^2)
reference Ewald2D) is out of this hot path's scope and raises.
Host numpy forms of ``langevin_step`` / ``nose_hoover_step`` /
``maxwell_velocities`` / ``kinetic_energy`` are kept for API compatibility.
"""

from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np

from .core import BoxGeometry, EwaldParams, ParticleSystem, choose_alpha, make_ewald_params
from .ewald2d import check_short_range_cutoff, raise_on_status
from .rbse2d import ModeSampler, _rb_commonv, charge_term_sum, normalization_H
from .soe import SOEApprox, build_soe_contour
from .soewald2d import full_sum_constants

WCA_CUT = 2.0 ** (1.0 / 6.0)


def _status_errors(status: int, where: str) -> None:
    from ._native import SLAB_STATUS_COINCIDENT, SLAB_STATUS_WALL
    if status & SLAB_STATUS_WALL:
        raise ValueError("particle at or beyond a wall")
    if where == "lj" and status & SLAB_STATUS_COINCIDENT:
        raise ValueError("coincident particles in the repulsive core")
    raise_on_status(status)


def lj_forces(system: ParticleSystem, box: BoxGeometry, eps: float = 1.0, sigma: float = 1.0):
    """Purely repulsive pair core 4 eps [(s/r)^12 - (s/r)^6] + eps below
    r = 2^(1/6) s (md.py:34-56), on device.  Returns (energy, forces)."""
    n = system.n
    if n < 2 or eps == 0.0:
        return 0.0, np.zeros((n, 3))
    from .engine import get_engine, host_result, to_device
    import torch
    eng = get_engine()
    pos = to_device(system.pos)
    forces = torch.zeros((n, 3), dtype=torch.float64, device=eng.device)
    energy = torch.zeros(8, dtype=torch.float64, device=eng.device)
    while True:
        status = torch.zeros(1, dtype=torch.int32, device=eng.device)
        forces.zero_()
        eng.wca(pos, box, eps, sigma, forces, energy, status)
        st = int(status.cpu().item())
        if not eng.handle_overflow(st):
            break
    _status_errors(st, "lj")
    e, f = host_result(energy, forces)
    return float(e[0]), f


def wall_forces(system: ParticleSystem, box: BoxGeometry, eps: float = 1.0, sigma: float = 0.5):
    """The same repulsive form on the distances to z = 0 and z = lz (md.py:59-77)."""
    n = system.n
    if n == 0:
        return 0.0, np.zeros((0, 3))
    from .engine import get_engine, host_result, to_device
    import torch
    eng = get_engine()
    pos = to_device(system.pos)
    forces = torch.zeros((n, 3), dtype=torch.float64, device=eng.device)
    energy = torch.zeros(8, dtype=torch.float64, device=eng.device)
    status = torch.zeros(1, dtype=torch.int32, device=eng.device)
    eng.walls(pos, box.lz, eps, sigma, forces, energy, status)
    _status_errors(int(status.cpu().item()), "walls")
    e, f = host_result(energy, forces)
    return float(e[0]), f


@dataclass
class MDOptions:
    """Knobs for run_simulation; defaults give a stable dilute slab run (md.py:80-101)."""

    dt: float = 0.005
    n_steps: int = 1000
    equilibration: int = 0
    temperature: float = 1.0
    thermostat: str = "langevin"      # langevin | nose-hoover | none
    gamma: float = 1.0
    tau: float = 0.5
    solver: str = "soewald2d"         # soewald2d | rbse2d  (ewald2d: out of scope)
    alpha: float | None = None
    s: float = 4.0
    soe_size: int = 8
    batch_size: int = 16
    lj_eps: float = 1.0
    lj_sigma: float = 1.0
    wall_eps: float = 1.0
    wall_sigma: float = 0.5
    coulomb: bool = True
    seed: int = 0
    sample_every: int = 10


@dataclass
class MDResult:
    times: np.ndarray
    positions: np.ndarray             # wrapped, (n_samples, N, 3)
    unwrapped: np.ndarray             # (n_samples, N, 3), xy never wrapped
    velocities: np.ndarray
    potential: np.ndarray
    kinetic: np.ndarray
    conserved: np.ndarray             # NVE / NH invariant; nan for Langevin
    charge: np.ndarray
    mass: np.ndarray
    box: BoxGeometry
    options: MDOptions = field(repr=False)


class _ForceField:
    """Coulomb solver + WCA core + walls, evaluated on device (md.py:117-167).

    ``evaluate_device`` enqueues one evaluation into caller buffers: forces (N,3)
    and ``ebuf`` (10,) = [evaluate's 8 energy slots, u_lj, u_wall]; status bits
    are OR-ed into ``status``.  Nothing synchronises."""

    def __init__(self, box: BoxGeometry, charge: np.ndarray, opts: MDOptions, rb_seed: int):
        self.box = box
        self.opts = opts
        self.params: EwaldParams | None = None
        self.soe: SOEApprox | None = None
        self.sampler = None
        self.H = None
        self.c_q = None
        self._cv = None
        self._uq = 0.0
        self._Q = float(np.sum(np.asarray(charge) ** 2))
        self._ewald = None
        if opts.coulomb:
            if opts.solver not in ("soewald2d", "rbse2d", "ewald2d"):
                raise ValueError(f"unknown solver {opts.solver!r}")
            alpha = opts.alpha
            if alpha is None:
                alpha = choose_alpha(len(charge), box,
                                     "linear" if opts.solver == "rbse2d" else "balanced",
                                     prefactor=0.8, s=opts.s)
            self.params = make_ewald_params(alpha, opts.s, box)
            check_short_range_cutoff(box, self.params.r_c)
            self.soe = build_soe_contour(opts.soe_size) if opts.solver != "ewald2d" else None
            Q = self._Q
            if opts.solver == "ewald2d":
                # the reference evaluates ref_energy_forces, which requires neutrality
                from .core import validate_neutrality
                ok, residual = validate_neutrality(
                    ParticleSystem(np.asarray(charge), np.ones(len(charge)),
                                   np.zeros((len(charge), 3)), np.zeros((len(charge), 3))), box)
                if not ok:
                    raise ValueError(f"system is not charge neutral (residual {residual:g})")
            elif opts.solver == "rbse2d":
                self.sampler = ModeSampler(alpha, box, seed=rb_seed)
                self.H = normalization_H(alpha, box)
                self.c_q = charge_term_sum(alpha, box, Q)
            else:
                self._cv, self._uq = full_sum_constants(self.params, box, Q)
        self._dev = None

    def _device_consts(self, eng):
        if self._dev is None:
            from .engine import _SOEPack, to_device
            d = {}
            if self.opts.coulomb and self.opts.solver == "ewald2d":
                from .ewald2d import Ewald2DDevice
                self._ewald = Ewald2DDevice(eng, self.params, self.box, self._Q)
            elif self.opts.coulomb:
                d["pack"] = _SOEPack(self.soe)
                if self.opts.solver == "soewald2d":
                    km = self.params.kmodes
                    d["modes"] = to_device(km) if km.shape[0] else None
                    d["cv"] = to_device(self._cv) if km.shape[0] else 0.0
            self._dev = d
        return self._dev

    def evaluate_device(self, eng, pos, q, forces, ebuf, status):
        import torch
        opts = self.opts
        dev = self._device_consts(eng)
        if opts.coulomb and opts.solver == "ewald2d":
            self._ewald.enqueue(pos, q, forces, ebuf[:8], status)
        elif opts.coulomb:
            if opts.solver == "soewald2d":
                modes, cv, cconst = dev["modes"], dev["cv"], self._uq
            else:
                P = opts.batch_size
                modes = self.sampler.batch_device(P)
                cv, cconst = _rb_commonv(self.H, P, self.params.alpha), self.c_q
            eng.evaluate(pos, q, self.box, self.params.alpha, self.params.r_c, self.soe, modes,
                         cv, cconst, forces=forces, energy=ebuf[:8], soe_pack=dev["pack"])
            status.bitwise_or_(ebuf[5:6].to(torch.int32))
        else:
            forces.zero_()
            ebuf[:8].zero_()
        if opts.lj_eps:
            eng.wca(pos, self.box, opts.lj_eps, opts.lj_sigma, forces, ebuf[8:9], status)
        else:
            ebuf[8:9].zero_()
        eng.walls(pos, self.box.lz, opts.wall_eps, opts.wall_sigma, forces, ebuf[9:10], status)

    @staticmethod
    def total(e: np.ndarray) -> float:
        # EnergyBreakdown.total + u_lj + u_wall
        return float(e[0] + e[1] + e[2] - e[3] + e[4] + e[8] + e[9])

    def evaluate(self, system: ParticleSystem):
        """Host form of md.py:144-167: (potential energy, forces (N,3))."""
        from .engine import get_engine, host_result, to_device
        import torch
        eng = get_engine()
        pos, q = to_device(system.pos), to_device(system.charge)
        n = system.n
        while True:
            forces = torch.zeros((n, 3), dtype=torch.float64, device=eng.device)
            ebuf = torch.zeros(10, dtype=torch.float64, device=eng.device)
            status = torch.zeros(1, dtype=torch.int32, device=eng.device)
            self.evaluate_device(eng, pos, q, forces, ebuf, status)
            e, f = host_result(ebuf, forces)
            st = int(status.cpu().item())
            if not eng.handle_overflow(st):
                break
        _status_errors(st, "lj")
        return self.total(e), f


def maxwell_velocities(mass: np.ndarray, temperature: float,
                       rng: np.random.Generator) -> np.ndarray:
    """Initial velocities as md.py:170-174 draws them: Gaussian components of
    variance T / m, then the centre-of-mass momentum removed (host, once per run)."""
    m = np.asarray(mass, dtype=np.float64)
    scale = np.sqrt(temperature / m)
    v = rng.normal(size=(m.size, 3)) * scale[:, None]
    p_com = m @ v                     # total momentum (3,)
    return v - p_com[None, :] / m.sum()


def kinetic_energy(mass: np.ndarray, vel: np.ndarray) -> float:
    """sum_i m_i |v_i|^2 / 2 (md.py:176-177); the device form is slab_md_kinetic."""
    return 0.5 * float(np.einsum("i,ij,ij->", mass, vel, vel))


def langevin_step(pos, vel, forces, mass, dt, gamma, temperature, noise):
    """Host reference of the device BAOAB step (slab_md_langevin; md.py:180-193):
    half kick (B), half drift (A), exact Ornstein-Uhlenbeck update (O) with the
    caller's standard-normal ``noise``, half drift (A).  No x, y wrap here."""
    m = np.asarray(mass, dtype=np.float64)[:, None]
    half = 0.5 * dt
    decay = np.exp(-gamma * dt)
    v = vel + half * forces / m                                            # B
    x = pos + half * v                                                     # A
    v = decay * v + np.sqrt((1.0 - decay * decay) * temperature / m) * noise  # O
    return x + half * v, v                                                 # A


def run_simulation(system: ParticleSystem, box: BoxGeometry, opts: MDOptions) -> MDResult:
    """Integrate and sample (md.py:227-325) with device-resident state: per step
    only kernel launches; the host reads energies / positions at sample points."""
    from .engine import get_engine, to_device
    import torch
    n = system.n
    if opts.thermostat not in ("langevin", "nose-hoover", "none"):
        raise ValueError(f"unknown thermostat {opts.thermostat!r}")
    eq = opts.equilibration
    if not 0 <= eq <= opts.n_steps:
        raise ValueError("equilibration must lie in [0, n_steps]")
    ss = np.random.SeedSequence(opts.seed)
    thermo_ss, rb_ss, vel_ss = ss.spawn(3)
    ff = _ForceField(box, system.charge, opts, rb_seed=int(rb_ss.generate_state(1)[0]))
    thermo_seed = int(thermo_ss.generate_state(1, dtype=np.uint64)[0])
    mass_h = np.asarray(system.mass, dtype=np.float64)
    if system.vel is not None and np.any(system.vel):
        vel_h = np.array(system.vel, dtype=np.float64)
    else:
        vel_h = maxwell_velocities(mass_h, opts.temperature,
                                   np.random.Generator(np.random.Philox(vel_ss)))
    eng = get_engine()
    dev = eng.device
    pos = to_device(system.pos).clone()
    vel = to_device(vel_h).clone()
    q = to_device(system.charge)
    mass = to_device(mass_h)
    shift = torch.zeros((n, 2), dtype=torch.float64, device=dev)
    forces = torch.zeros((n, 3), dtype=torch.float64, device=dev)
    ebuf = torch.zeros(10, dtype=torch.float64, device=dev)
    status = torch.zeros(1, dtype=torch.int32, device=dev)
    counter = torch.zeros(1, dtype=torch.int64, device=dev)
    kin = torch.zeros(1, dtype=torch.float64, device=dev)
    dt = opts.dt

    eng.md_drift(pos, vel, 0.0, shift, box)  # initial wrap (md.py:255)

    def evaluate():
        ff.evaluate_device(eng, pos, q, forces, ebuf, status)

    # first evaluation: settle the neighbour capacity (may rerun once)
    while True:
        status.zero_()
        evaluate()
        st = int(status.cpu().item())
        if not eng.handle_overflow(st):
            break
    _status_errors(st, "lj")

    n_samples = (opts.n_steps - eq) // opts.sample_every + 1
    times = np.empty(n_samples)
    traj = np.empty((n_samples, n, 3))
    traj_un = np.empty((n_samples, n, 3))
    vels = np.empty((n_samples, n, 3))
    pot = np.empty(n_samples)
    kin_h = np.empty(n_samples)
    cons = np.full(n_samples, np.nan)
    xi = 0.0
    eta = 0.0
    n_f = 3 * n
    q_nh = n_f * opts.temperature * opts.tau ** 2

    def kinetic():
        eng.md_kinetic(vel, mass, kin)
        return float(kin.cpu().item())

    def record(idx, step):
        st_ = int(status.cpu().item())
        if st_:
            _status_errors(st_, "lj")
            # a row overflow was evaluated in-stream (complete results): only
            # grow the capacity for the steps that follow
            eng.handle_overflow(st_)
        e = ebuf.cpu().numpy()
        p = pos.cpu().numpy()
        sh = shift.cpu().numpy()
        times[idx] = step * dt
        traj[idx] = p
        traj_un[idx] = p
        traj_un[idx, :, 0] += sh[:, 0]
        traj_un[idx, :, 1] += sh[:, 1]
        vels[idx] = vel.cpu().numpy()
        u_now = _ForceField.total(e)
        pot[idx] = u_now
        kin_h[idx] = kinetic()
        if opts.thermostat == "none":
            cons[idx] = u_now + kin_h[idx]
        elif opts.thermostat == "nose-hoover":
            cons[idx] = u_now + kin_h[idx] + 0.5 * q_nh * xi ** 2 + n_f * opts.temperature * eta

    def nh_half():
        nonlocal xi, eta
        k2 = 2.0 * kinetic()
        xi += 0.25 * dt * (k2 - n_f * opts.temperature) / q_nh
        s = np.exp(-0.5 * dt * xi)
        eng.md_scale(vel, s)
        eta += 0.5 * dt * xi
        k2 = 2.0 * kinetic()
        xi += 0.25 * dt * (k2 - n_f * opts.temperature) / q_nh

    sample = 0
    if eq == 0:
        record(0, 0)
        sample = 1
    for step in range(1, opts.n_steps + 1):
        if opts.thermostat == "langevin":
            eng.md_langevin(pos, vel, forces, mass, dt, opts.gamma, opts.temperature,
                            thermo_seed, counter, shift, box)
            evaluate()
            eng.md_kick(vel, forces, mass, 0.5 * dt)
        elif opts.thermostat == "nose-hoover":
            nh_half()
            eng.md_kick(vel, forces, mass, 0.5 * dt)
            eng.md_drift(pos, vel, dt, shift, box)
            evaluate()
            eng.md_kick(vel, forces, mass, 0.5 * dt)
            nh_half()
        else:
            eng.md_kick(vel, forces, mass, 0.5 * dt)
            eng.md_drift(pos, vel, dt, shift, box)
            evaluate()
            eng.md_kick(vel, forces, mass, 0.5 * dt)
        if step >= eq and (step - eq) % opts.sample_every == 0:
            record(sample, step)
            sample += 1

    return MDResult(times=times, positions=traj, unwrapped=traj_un, velocities=vels,
                    potential=pot, kinetic=kin_h, conserved=cons,
                    charge=np.array(system.charge, dtype=np.float64), mass=mass_h.copy(),
                    box=box, options=opts)


# ---------------------------------------------------------------------------
# observables (host, post-processing of the sampled frames; md.py:332-376)
# ---------------------------------------------------------------------------
def _msd_at_lags(unwrapped: np.ndarray, lags: np.ndarray):
    """Multiple-time-origin mean-square displacement at each lag, split into the
    in-plane (x, y) and normal (z) parts."""
    out_xy = np.empty(lags.size)
    out_z = np.empty(lags.size)
    for k, lag in enumerate(lags):
        disp = unwrapped[lag:] - unwrapped[:-lag]          # (origins, n, 3)
        sq = disp * disp
        out_xy[k] = (sq[..., 0] + sq[..., 1]).mean()
        out_z[k] = sq[..., 2].mean()
    return out_xy, out_z


def _z_profiles(z_frames: np.ndarray, charge: np.ndarray, lz: float, area: float,
                n_bins: int, n_blocks: int):
    """Number density per charge species in n_bins z slabs, averaged within each
    of n_blocks contiguous frame blocks; (mean, sample std) over the blocks."""
    width = lz / n_bins
    # slab index of every (frame, particle); z == lz belongs to the top slab
    slab = np.minimum((z_frames / width).astype(np.int64), n_bins - 1)
    slab = np.maximum(slab, 0)
    blocks = np.array_split(np.arange(z_frames.shape[0]), n_blocks)
    mean, std = {}, {}
    for sp in np.unique(charge):
        cols = np.flatnonzero(charge == sp)
        per_block = np.stack([
            np.bincount(slab[blk][:, cols].ravel(), minlength=n_bins)[:n_bins]
            / (blk.size * area * width) for blk in blocks])
        mean[float(sp)] = per_block.mean(axis=0)
        std[float(sp)] = per_block.std(axis=0, ddof=1)
    return mean, std


def compute_observables(result: MDResult, n_bins: int = 40, n_blocks: int = 5,
                        max_lag_frac: float = 0.5, skip_frac: float = 0.2) -> dict:
    """The reference's trajectory observables (md.py:332-376): MSDs over the
    frames after the first ``skip_frac`` (lags up to ``max_lag_frac`` of them, at
    most 60 distinct values) and block-averaged z concentration profiles."""
    frames = len(result.times)
    first = int(skip_frac * frames)
    unwrapped = result.unwrapped[first:]
    kept = unwrapped.shape[0]
    if kept < 4:
        raise ValueError("trajectory too short for observables")
    dt_frame = result.times[1] - result.times[0] if frames > 1 else 1.0
    lag_max = max(1, int(max_lag_frac * kept))
    lags = np.unique(np.linspace(1, lag_max, min(60, lag_max)).astype(int))
    msd_xy, msd_z = _msd_at_lags(unwrapped, lags)
    box = result.box
    conc, conc_std = _z_profiles(result.positions[first:, :, 2], np.asarray(result.charge),
                                 box.lz, box.area, n_bins, n_blocks)
    centers = (np.arange(n_bins) + 0.5) * (box.lz / n_bins)
    return {"lag_times": lags * dt_frame, "msd_xy": msd_xy, "msd_z": msd_z,
            "z_bin_centers": centers, "concentration": conc, "concentration_std": conc_std}
