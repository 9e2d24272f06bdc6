"""Device-side engine: torch owns device memory and streams, the C-ABI does the work.

``Engine`` wraps one ``SlabCtx`` per CUDA device.  Its methods take torch CUDA
tensors and enqueue C-ABI calls on the current torch stream; they never fall
back to the CPU.  ``DeviceEvaluator`` keeps a whole RBSE2D / SOEwald2D step
device-resident (positions, sampled modes, forces, energies) and can replay it
as a CUDA graph -- the form the MD loop and ``bench.py`` use.
"""

from __future__ import annotations

import ctypes
import math

import numpy as np

from . import _native
from ._native import SlabBox, SlabEvalArgs, SlabSOE, check

_engines: dict = {}


def _torch():
    import torch
    return torch


def require_cuda():
    torch = _torch()
    if not torch.cuda.is_available():
        raise _native.NativeUnavailable(
            "no CUDA device visible: this package has no CPU fallback")
    _native.load()
    return torch


class _SOEPack:
    """Host copies of the SOE table kept alive for the duration of a call."""

    def __init__(self, soe):
        w = np.asarray(soe.w, dtype=np.complex128)
        s = np.asarray(soe.s, dtype=np.complex128)
        self.arrays = [np.ascontiguousarray(a) for a in (w.real, w.imag, s.real, s.imag)]
        p = [a.ctypes.data_as(ctypes.POINTER(ctypes.c_double)) for a in self.arrays]
        self.struct = SlabSOE(len(w), *p)


def _ptr(t):
    return None if t is None else ctypes.c_void_p(t.data_ptr())


class Engine:
    def __init__(self, device):
        torch = require_cuda()
        self.device = torch.device(device)
        self.lib = _native.load()
        self.ctx = ctypes.c_void_p()
        with torch.cuda.device(self.device):
            check(self.lib.slab_ctx_create(ctypes.byref(self.ctx)), "slab_ctx_create")

    def handle_overflow(self, status: int) -> bool:
        """After a synchronised run: if a short-range neighbour row overflowed, grow the
        capacity to the longest row seen, so that later runs keep every home on the
        row path.  Returns False: the overflowed homes were already evaluated
        in-stream by the overflow kernel (short.cu), the results are complete and
        nothing needs to be rerun -- a device-resident / graph-replayed step never
        drops a pair, whatever the local density does between host checks."""
        if not int(status) & _native.SLAB_STATUS_NBR_OVERFLOW:
            return False
        need = ctypes.c_int(0)
        check(self.lib.slab_ctx_last_max_neighbors(self.ctx, ctypes.byref(need)),
              "slab_ctx_last_max_neighbors")
        check(self.lib.slab_ctx_neighbor_capacity(self.ctx, int(need.value * 1.1) + 16),
              "slab_ctx_neighbor_capacity")
        return False

    def _stream(self):
        torch = _torch()
        return ctypes.c_void_p(torch.cuda.current_stream(self.device).cuda_stream)

    # -- sort ---------------------------------------------------------------
    def sort_by_z(self, z, stride: int = 1):
        torch = _torch()
        n = z.numel() // stride if stride > 1 else z.numel()
        perm = torch.empty(n, dtype=torch.int64, device=self.device)
        check(self.lib.slab_sort_by_z(self.ctx, _ptr(z), stride, n, _ptr(perm), self._stream()),
              "slab_sort_by_z")
        return perm

    # -- full evaluation ----------------------------------------------------
    def evaluate(self, pos, charge, box, alpha, r_c, soe, modes, commonv, charge_const,
                 forces=None, energy=None, want_forces=True, skip_short_range=False,
                 perm=None, soe_pack=None, shard=(0, 1), scan_events=None, shard_mode=0,
                 phase=0, xchg=None, modes_ready=None):
        """Enqueue one energy/force evaluation.  ``commonv`` is a float (RB) or a
        (P,) device tensor (full mode sum).  Writes energy (8,) and forces (n,3).

        ``shard=(rank, count)``: multi-GPU share (caller passes this rank's mode
        slice and sums forces / energy[0:5] over ranks).  ``scan_events``: a pair
        of torch.cuda.Event recorded around the SOE scan kernels.
        ``shard_mode=1`` (z-split): ``phase`` 1 writes this rank's exchange payload
        into ``xchg``, phase 2 (``xchg`` = all ranks' payloads, rank order)
        finishes; see ``SlabEvalArgs`` in the header."""
        torch = _torch()
        n = charge.numel()
        if energy is None:
            energy = torch.empty(8, dtype=torch.float64, device=self.device)
        if forces is None and want_forces:
            forces = torch.empty((n, 3), dtype=torch.float64, device=self.device)
        pack = soe_pack or _SOEPack(soe)
        P = 0 if modes is None else modes.shape[0]
        cv_t = commonv if torch.is_tensor(commonv) else None
        args = SlabEvalArgs(
            n=n, d_pos=_ptr(pos), d_charge=_ptr(charge),
            box=SlabBox(box.lx, box.ly, box.lz, box.sigma_top, box.sigma_bot),
            alpha=float(alpha), r_c=float(r_c), soe=pack.struct,
            d_modes=_ptr(modes) if P else None, nmode=P, d_commonv=_ptr(cv_t),
            commonv_scalar=0.0 if cv_t is not None else float(commonv),
            charge_const=float(charge_const), want_forces=1 if want_forces else 0,
            skip_short_range=1 if skip_short_range else 0,
            d_forces=_ptr(forces) if want_forces else None, d_energy=_ptr(energy),
            d_perm=_ptr(perm), shard_rank=int(shard[0]), shard_count=int(shard[1]),
            ev_scan_begin=ctypes.c_void_p(scan_events[0].cuda_event) if scan_events else None,
            ev_scan_end=ctypes.c_void_p(scan_events[1].cuda_event) if scan_events else None,
            shard_mode=int(shard_mode), phase=int(phase), d_xchg=_ptr(xchg),
            ev_modes_ready=ctypes.c_void_p(modes_ready.cuda_event) if modes_ready else None)
        check(self.lib.slab_evaluate(self.ctx, ctypes.byref(args), self._stream()),
              "slab_evaluate")
        return energy, forces

    def evaluate_host(self, pos, charge, box, alpha, r_c, soe, modes, commonv, charge_const,
                      want_forces=True, skip_short_range=False):
        """One evaluation on HOST arrays through ``slab_evaluate_host`` (uploads on
        a side stream, charges overlapping the z sort; one synchronisation).
        ``pos`` (n,3) / ``charge`` (n,) float64 numpy (page-locked memory copies at
        DMA speed); ``modes`` a device (P,3) tensor or None; returns numpy
        (energy (8,), forces (n,3) or None) backed by page-locked buffers."""
        torch = _torch()
        pos = np.ascontiguousarray(pos, dtype=np.float64)
        charge = np.ascontiguousarray(charge, dtype=np.float64)
        n = charge.shape[0]
        if pos.shape != (n, 3):
            raise ValueError("pos must be (n, 3)")
        e_h = torch.empty(8, dtype=torch.float64, pin_memory=True)
        f_h = torch.empty((n, 3), dtype=torch.float64, pin_memory=True) if want_forces else None
        pack = _SOEPack(soe)
        P = 0 if modes is None else modes.shape[0]
        cv_t = commonv if torch.is_tensor(commonv) else None
        args = SlabEvalArgs(
            n=n, box=SlabBox(box.lx, box.ly, box.lz, box.sigma_top, box.sigma_bot),
            alpha=float(alpha), r_c=float(r_c), soe=pack.struct,
            d_modes=_ptr(modes) if P else None, nmode=P, d_commonv=_ptr(cv_t),
            commonv_scalar=0.0 if cv_t is not None else float(commonv),
            charge_const=float(charge_const), want_forces=1 if want_forces else 0,
            skip_short_range=1 if skip_short_range else 0, shard_rank=0, shard_count=1,
            shard_mode=0, phase=0)
        hp = ctypes.c_void_p
        check(self.lib.slab_evaluate_host(
            self.ctx, ctypes.byref(args), hp(pos.ctypes.data), hp(charge.ctypes.data),
            _ptr(f_h), _ptr(e_h), self._stream()), "slab_evaluate_host")
        return e_h.numpy(), (f_h.numpy() if f_h is not None else None)

    # -- sub-paths ----------------------------------------------------------
    def short_range(self, pos, charge, box, alpha, r_c):
        """Synchronous: (energy, forces, status), rerun once after a capacity overflow."""
        while True:
            out = self._short_range(pos, charge, box, alpha, r_c)
            if not self.handle_overflow(int(out[2].cpu().item())):
                return out

    def _short_range(self, pos, charge, box, alpha, r_c):
        torch = _torch()
        n = charge.numel()
        forces = torch.empty((n, 3), dtype=torch.float64, device=self.device)
        energy = torch.zeros(1, dtype=torch.float64, device=self.device)
        status = torch.zeros(1, dtype=torch.int32, device=self.device)
        check(self.lib.slab_short_range(
            self.ctx, _ptr(pos), _ptr(charge), n,
            SlabBox(box.lx, box.ly, box.lz, box.sigma_top, box.sigma_bot), float(alpha),
            float(r_c), _ptr(forces), _ptr(energy), _ptr(status), self._stream()),
            "slab_short_range")
        return energy, forces, status

    def fourier_sweep(self, x, y, z, q, modes, commonv, soe, alpha, area, want_forces,
                      forces_sorted=None):
        torch = _torch()
        n = q.numel()
        energy = torch.zeros(1, dtype=torch.float64, device=self.device)
        status = torch.zeros(1, dtype=torch.int32, device=self.device)
        pack = _SOEPack(soe)
        cv_t = commonv if torch.is_tensor(commonv) else None
        check(self.lib.slab_fourier_sweep(
            self.ctx, _ptr(x), _ptr(y), _ptr(z), _ptr(q), n, _ptr(modes), _ptr(cv_t),
            0.0 if cv_t is not None else float(commonv), modes.shape[0], pack.struct,
            float(alpha), float(area), 1 if want_forces else 0, _ptr(forces_sorted),
            _ptr(energy), _ptr(status), self._stream()), "slab_fourier_sweep")
        return energy, status

    def zero_mode_sweep(self, z, q, soe, alpha, want_forces, fz=None):
        torch = _torch()
        energy = torch.zeros(1, dtype=torch.float64, device=self.device)
        pack = _SOEPack(soe)
        check(self.lib.slab_zero_mode_sweep(
            self.ctx, _ptr(z), _ptr(q), q.numel(), pack.struct, float(alpha),
            1 if want_forces else 0, _ptr(fz), _ptr(energy), self._stream()),
            "slab_zero_mode_sweep")
        return energy

    def sample_modes(self, state, seed, alpha, lx, ly, thin, burn_in, P, modes=None, idx=None):
        check(self.lib.slab_sample_modes(
            self.ctx, _ptr(state), ctypes.c_uint64(seed), float(alpha), float(lx), float(ly),
            int(thin), int(burn_in), int(P), _ptr(modes), _ptr(idx), self._stream()),
            "slab_sample_modes")

    def batch_energies(self, pos, charge, soe, alpha, area, modes, nbatch, P, commonv):
        """Forward-sweep energies of nbatch consecutive P-mode batches (device (nbatch,)
        tensor) and the status word (device int32)."""
        torch = _torch()
        out = torch.empty(nbatch, dtype=torch.float64, device=self.device)
        status = torch.zeros(1, dtype=torch.int32, device=self.device)
        pack = _SOEPack(soe)
        check(self.lib.slab_batch_energies(
            self.ctx, _ptr(pos), _ptr(charge), charge.numel(), pack.struct, float(alpha),
            float(area), _ptr(modes), int(nbatch), int(P), float(commonv), _ptr(out),
            _ptr(status), self._stream()), "slab_batch_energies")
        return out, status

    # -- MD step (md.cu) ------------------------------------------------------
    def wca(self, pos, box, eps, sigma, forces, energy, status):
        """Enqueue: forces += WCA core forces; energy[0] = WCA energy; status |= bits."""
        check(self.lib.slab_wca(
            self.ctx, _ptr(pos), pos.shape[0],
            SlabBox(box.lx, box.ly, box.lz, box.sigma_top, box.sigma_bot), float(eps),
            float(sigma), _ptr(forces), _ptr(energy), _ptr(status), self._stream()), "slab_wca")

    def walls(self, pos, lz, eps, sigma, forces, energy, status):
        check(self.lib.slab_walls(self.ctx, _ptr(pos), pos.shape[0], float(lz), float(eps),
                                  float(sigma), _ptr(forces), _ptr(energy), _ptr(status),
                                  self._stream()), "slab_walls")

    def md_langevin(self, pos, vel, forces, mass, dt, gamma, temperature, seed, counter, shift,
                    box):
        check(self.lib.slab_md_langevin(
            _ptr(pos), _ptr(vel), _ptr(forces), _ptr(mass), pos.shape[0], float(dt), float(gamma),
            float(temperature), ctypes.c_uint64(int(seed) & 0xFFFFFFFFFFFFFFFF), _ptr(counter),
            _ptr(shift), float(box.lx), float(box.ly), self._stream()), "slab_md_langevin")

    def md_kick(self, vel, forces, mass, h):
        check(self.lib.slab_md_kick(_ptr(vel), _ptr(forces), _ptr(mass), vel.shape[0], float(h),
                                    self._stream()), "slab_md_kick")

    def md_drift(self, pos, vel, dt, shift, box):
        check(self.lib.slab_md_drift(_ptr(pos), _ptr(vel), pos.shape[0], float(dt), _ptr(shift),
                                     float(box.lx), float(box.ly), self._stream()),
              "slab_md_drift")

    def md_scale(self, vel, s):
        check(self.lib.slab_md_scale(_ptr(vel), vel.shape[0], float(s), self._stream()),
              "slab_md_scale")

    def md_kinetic(self, vel, mass, out):
        check(self.lib.slab_md_kinetic(self.ctx, _ptr(vel), _ptr(mass), vel.shape[0], _ptr(out),
                                       self._stream()), "slab_md_kinetic")

    def constant_terms(self, pos, charge, box, alpha):
        """Device (8,) energy vector with u_self (slot 3) and u_ps (slot 4) from the
        assembly's own reduction."""
        torch = _torch()
        energy = torch.zeros(8, dtype=torch.float64, device=self.device)
        check(self.lib.slab_constant_terms(
            self.ctx, _ptr(pos), _ptr(charge), charge.numel(),
            SlabBox(box.lx, box.ly, box.lz, box.sigma_top, box.sigma_bot), float(alpha),
            _ptr(energy), self._stream()), "slab_constant_terms")
        return energy

    def recursive_pair_sum(self, q, theta, z, beta):
        torch = _torch()
        out = torch.empty((q.numel(), 2), dtype=torch.float64, device=self.device)
        check(self.lib.slab_recursive_pair_sum(
            self.ctx, _ptr(q), _ptr(theta), _ptr(z), q.numel(), float(beta.real),
            float(beta.imag), _ptr(out), self._stream()), "slab_recursive_pair_sum")
        return out


def get_engine(device=None) -> Engine:
    torch = require_cuda()
    dev = torch.device(device if device is not None else f"cuda:{torch.cuda.current_device()}")
    if dev.index is None:
        dev = torch.device(f"cuda:{torch.cuda.current_device()}")
    eng = _engines.get(dev.index)
    if eng is None:
        eng = _engines[dev.index] = Engine(dev)
    return eng


def to_device(a, dtype=None, device=None):
    """Host array -> device tensor.  Memory that is already page-locked (e.g. a
    numpy view of a pinned torch buffer) is copied asynchronously by DMA."""
    torch = require_cuda()
    eng = get_engine(device)
    t = torch.as_tensor(np.ascontiguousarray(a), dtype=dtype or torch.float64)
    return t.to(eng.device, non_blocking=t.is_pinned())


_pinned_keepalive: list = []


def host_result(energy, forces=None):
    """Device energy (8,) and forces (n,3) -> numpy, through page-locked buffers from
    torch's caching host allocator (one synchronisation, DMA-speed copies).  The
    returned arrays own their buffers (freed back to the cache when dropped)."""
    torch = _torch()
    e_h = torch.empty(energy.shape, dtype=energy.dtype, pin_memory=True)
    e_h.copy_(energy, non_blocking=True)
    f_h = None
    if forces is not None:
        f_h = torch.empty(forces.shape, dtype=forces.dtype, pin_memory=True)
        f_h.copy_(forces, non_blocking=True)
    torch.cuda.current_stream(energy.device).synchronize()
    return e_h.numpy(), (f_h.numpy() if f_h is not None else None)


def pinned_like(a) -> np.ndarray:
    """A numpy array backed by pinned (page-locked) host memory, filled with `a`
    (the backing torch buffer is kept alive for the life of the process)."""
    torch = require_cuda()
    a = np.ascontiguousarray(a, dtype=np.float64)
    buf = torch.empty(a.shape, dtype=torch.float64, pin_memory=True)
    _pinned_keepalive.append(buf)
    out = buf.numpy()
    out[...] = a
    return out


def device_sort_perm(z: np.ndarray, lz: float) -> np.ndarray:
    """Host helper behind core.sort_by_z: device radix sort, permutation to numpy."""
    eng = get_engine()
    torch = _torch()
    if z.size == 0:
        return np.zeros(0, dtype=np.int64)
    zt = torch.as_tensor(np.ascontiguousarray(z, dtype=np.float64)).to(eng.device)
    perm = eng.sort_by_z(zt, 1)
    return perm.cpu().numpy()


class DeviceEvaluator:
    """A device-resident RBSE2D (``P`` sampled modes) or SOEwald2D (full mode set) step.

    Positions / charges live on the device; each ``step()`` (optionally) draws a
    fresh k-set with the device sampler and evaluates energy + forces, all on one
    stream with no host synchronisation.  ``capture()`` records the step as a
    CUDA graph so small systems are not launch bound.

    Multi-GPU (``world > 1``, one process per GPU): particles are
    replicated, every rank draws the SAME k-set (same seed, counter-based
    stream), evaluates its contiguous slice of the modes plus its share of the
    short-range home particles (rank 0 adds the k = 0 mode and the constants),
    and the partial forces + energies -- one packed (3N + 8) fp64 buffer -- are
    combined with ONE all-reduce (NCCL over NVLink).
    """

    def __init__(self, system, box, params, soe, P=None, H=None, c_q=None, seed=0, thin=10,
                 burn_in=100, modes=None, device=None, sample=True, rank=0, world=1,
                 group=None, shard_mode="modes"):
        from .rbse2d import charge_term_sum, normalization_H
        from .soewald2d import full_sum_constants
        torch = require_cuda()
        self.eng = get_engine(device)
        dev = self.eng.device
        self.box, self.params, self.soe = box, params, soe
        self.alpha = params.alpha
        self.pack = _SOEPack(soe)
        self.n = system.n
        self.rank, self.world, self.group = int(rank), int(world), group
        self.reduce = self.world > 1  # one all-reduce of `packed` per step
        self.pos = torch.as_tensor(system.pos).to(dev)
        self.charge = torch.as_tensor(system.charge).to(dev)
        # forces and energies in one buffer: the multi-GPU path all-reduces it once
        self.packed = torch.zeros(3 * self.n + 8, dtype=torch.float64, device=dev)
        self.forces = self.packed[:3 * self.n].view(self.n, 3)
        self.energy = self.packed[3 * self.n:]
        self.graph = None
        self.graphs = []
        Q = float(np.sum(system.charge ** 2))
        if P is None:  # deterministic full mode sum (soe_energy_forces)
            self.P = params.kmodes.shape[0]
            cv, uq = full_sum_constants(params, box, Q)
            self.modes = torch.as_tensor(params.kmodes).to(dev)
            self.commonv = torch.as_tensor(cv).to(dev)
            self.charge_const = uq
            self.sample = False
        else:
            self.P = int(P)
            self.H = normalization_H(self.alpha, box) if H is None else H
            self.charge_const = charge_term_sum(self.alpha, box, Q) if c_q is None else c_q
            self.commonv = (self.H / self.P) * (2.0 / math.sqrt(math.pi)) * self.alpha
            self.modes = torch.empty((self.P, 3), dtype=torch.float64, device=dev)
            self.sample = sample and modes is None
            if modes is not None:
                self.modes.copy_(torch.as_tensor(np.asarray(modes, dtype=np.float64)))
            self.seed, self.thin = int(seed), int(thin)
            self.state = torch.zeros(6, dtype=torch.int64, device=dev)
            if self.sample:
                self.eng.sample_modes(self.state, self.seed, self.alpha, box.lx, box.ly,
                                      self.thin, burn_in, 0)
                # the chain for each step runs on a side stream, overlapping the
                # z sort; the evaluation waits on this event before the k-set's
                # first use
                self.side = torch.cuda.Stream(dev)
                self.ev_modes = torch.cuda.Event()
        # multi-GPU split: "modes" (default) -- each rank scans its
        # slice of the sampled modes over all particles, no mid-evaluation
        # exchange, ONE all-reduce per step; "zsplit" -- every rank scans all modes
        # over its contiguous range of the z-sorted particles, with an all-gather of
        # the chunk-range maps between the two phases
        if shard_mode not in ("zsplit", "modes"):
            raise ValueError("shard_mode must be 'zsplit' or 'modes'")
        self.zsplit = shard_mode == "zsplit" and self.world > 1
        from .sharding import mode_slice
        self.t0, self.t1 = (0, self.P) if self.zsplit else mode_slice(self.P, self.rank,
                                                                      self.world)
        if self.zsplit:
            cnt = int(_native.load().slab_zsplit_exchange_doubles(self.P, len(soe.w), 1))
            self.xloc = torch.zeros(max(cnt, 1), dtype=torch.float64, device=dev)
            self.xall = torch.zeros(self.world * max(cnt, 1), dtype=torch.float64, device=dev)

    def set_positions(self, pos):
        """Replace the device positions (e.g. after an MD update), in place."""
        self.pos.copy_(pos if hasattr(pos, "device") else
                       _torch().as_tensor(np.asarray(pos, dtype=np.float64)))

    def _enqueue_part(self, part, scan_events=None):
        """One rank's local work of a step: ``part`` "all" (single GPU or the
        "modes" split), "p1" / "p2" (the z-split phases around the exchange).
        No collective in here, so each part can be captured as a CUDA graph."""
        torch = _torch()
        ready = None
        if self.sample and part != "p2":
            # after everything queued so far (the previous step still reads the
            # k-set buffer), concurrently with this step's sort
            self.side.wait_stream(torch.cuda.current_stream(self.eng.device))
            with torch.cuda.stream(self.side):
                self.eng.sample_modes(self.state, self.seed, self.alpha, self.box.lx,
                                      self.box.ly, self.thin, 0, self.P, self.modes)
            self.ev_modes.record(self.side)
            ready = self.ev_modes
        modes = self.modes[self.t0:self.t1] if self.t1 > self.t0 else None
        cv = self.commonv[self.t0:self.t1] if torch.is_tensor(self.commonv) else self.commonv
        args = (self.pos, self.charge, self.box, self.alpha, self.params.r_c, self.soe, modes,
                cv, self.charge_const)
        kw = dict(forces=self.forces, energy=self.energy, soe_pack=self.pack,
                  shard=(self.rank, self.world), scan_events=scan_events)
        if part == "p1":
            self.eng.evaluate(*args, shard_mode=1, phase=1, xchg=self.xloc, modes_ready=ready,
                              **kw)
        elif part == "p2":
            self.eng.evaluate(*args, shard_mode=1, phase=2, xchg=self.xall, **kw)
        else:
            self.eng.evaluate(*args, modes_ready=ready, **kw)

    def _enqueue(self, scan_events=None):
        if self.zsplit:
            self._enqueue_part("p1", scan_events)
            self.exchange(self.xloc, self.xall)
            self._enqueue_part("p2", scan_events)
        else:
            self._enqueue_part("all", scan_events)
        if self.reduce:
            self.all_reduce(self.packed)

    def status(self) -> int:
        """Status bits of the last step (any rank, after the all-reduce); synchronous."""
        from .ewald2d import status_of
        return status_of(self.energy.cpu().numpy(), summed=self.reduce)

    def _host_staged(self) -> bool:
        """A gloo group (CPU tests, several processes sharing one GPU) takes its
        collectives through host copies; NCCL works on the device buffers."""
        import torch.distributed as dist
        return dist.get_backend(self.group) == "gloo"

    def all_reduce(self, buf):
        """Sum of the packed (forces, energies) buffer over ranks: the one
        collective of a "modes" step."""
        import torch.distributed as dist
        if self._host_staged():
            h = buf.cpu()
            dist.all_reduce(h, op=dist.ReduceOp.SUM, group=self.group)
            buf.copy_(h)
        else:
            dist.all_reduce(buf, op=dist.ReduceOp.SUM, group=self.group)

    def exchange(self, local, gathered):
        """z-split: every rank's chunk-range maps, in rank order (all-gather)."""
        import torch.distributed as dist
        if self._host_staged():
            h = gathered.cpu()
            dist.all_gather_into_tensor(h, local.cpu(), group=self.group)
            gathered.copy_(h)
        else:
            dist.all_gather_into_tensor(gathered, local, group=self.group)

    def warmup(self):
        """Run one step synchronously (workspace allocation, kernel attributes,
        short-range neighbour capacity)."""
        torch = _torch()
        while True:
            self._enqueue()
            torch.cuda.synchronize(self.eng.device)
            if not self.eng.handle_overflow(self.status()):
                return

    def capture(self, scan_events=None):
        """Record one step as a CUDA graph (small systems are launch bound).
        With ``scan_events`` (a pair of timing events, single GPU) the graph
        stamps them around the SOE scan on every replay and is returned without
        replacing the step's own graph (bench.py times the scan span inside the
        replayed step).  Multi-GPU: each rank's local parts are captured (the
        z-split phases as two graphs) and the collectives stay outside them, run
        between the replays by ``step``."""
        torch = _torch()
        if self.world > 1 and scan_events is not None:
            raise RuntimeError("scan-event graphs are single-GPU only")
        s = torch.cuda.Stream(self.eng.device)
        s.wait_stream(torch.cuda.current_stream(self.eng.device))
        with torch.cuda.stream(s):
            self.warmup()  # outside capture: workspace, func attributes
        torch.cuda.current_stream(self.eng.device).wait_stream(s)
        torch.cuda.synchronize(self.eng.device)
        parts = ("p1", "p2") if self.zsplit else ("all",)
        graphs = []
        for part in parts:
            g = torch.cuda.CUDAGraph()
            with torch.cuda.graph(g):
                if self.world > 1:
                    self._enqueue_part(part)
                else:
                    self._enqueue(scan_events)
            graphs.append(g)
        if scan_events is None:
            self.graph = graphs[0]
            self.graphs = graphs
        return graphs[0]

    def step(self, scan_events=None):
        if self.graph is not None and scan_events is None:
            if self.world == 1:
                self.graph.replay()
            else:
                self.graphs[0].replay()
                if self.zsplit:
                    self.exchange(self.xloc, self.xall)
                    self.graphs[1].replay()
                if self.reduce:
                    self.all_reduce(self.packed)
        else:
            self._enqueue(scan_events)
        return self.energy, self.forces
