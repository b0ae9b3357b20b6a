"""B200 execution backend: ``run_program`` for op_par_loop programs.

Drop-in for reference ``executor.py:707-729``: same ``BackendConfig`` field
names and validation style, same ``RunResult``, same post-conditions (mesh
frozen; every written dat visible through ``dat.fetch()`` / ``dat.data``;
reduction results in ``glob.buffer``; loops run in program order).  The
backend name is ``"cuda"`` — the only one this package has: every loop runs
as hand-written sm_100a kernels from ``libmeshloop_b200.so`` and there is no
CPU fallback (an unbound kernel raises :class:`ExecError`).

A program is compiled once into a native ``ml_program`` (loop descriptors
with device pointers, plans, functor ids, a globals arena) and then replayed
— eagerly with per-loop CUDA-event timing, or as one CUDA graph
(``BackendConfig(use_graph=True)``).  Reductions stay on the device between
loops, so a MIN computed by one loop can be READ by the next without a host
round trip; globals travel to the host once per program run.

``nranks > 1`` (or a multi-process launch) routes to the owner-compute
multi-GPU layer in :mod:`paper_1403_7209_b200.multigpu`.
"""
from __future__ import annotations

import ctypes as C
import os
import time
from collections import OrderedDict
from dataclasses import dataclass
from typing import Callable, Sequence

import numpy as np

from . import _native as N
from .core import (INC, MAX, MIN, READ, WRITE_MODES, ExecError, Global, Loop, Mesh, MeshError)
from .device import (dat_mirror, fold_eligible, gather_eligible, gather_mirror, map_mirror,
                     pfold_mirror, plan_mirror)
from .chain import chain_program
from .kernels import resolve_kernel
from .perf import PerfCollector, PerfRecord, b_alg, useful_bytes
from .plan import plan_for, plan_stats

__all__ = ["BackendConfig", "RunResult", "ExchangeTimeout", "reduce_global", "run_program",
           "run_loop", "compile_program", "CompiledProgram"]

_BACKENDS = ("cuda",)


class ExchangeTimeout(ExecError):
    """A rank waited longer than the configured bound for a halo message."""


SCHEDULES = ("auto", "gather", "pfold", "colour")

# "auto": primary fold when an element gathers many more indirect components
# than it increments (its neighbour rows are then read once per element instead
# of once per incidence, and the secondary slots are cheap), gather otherwise.
# Measured on B200 (profiles/README.md): vflux (92 read / 10 INC components per
# element) and iflux+vflux (126 / 10) are faster as pfold; iflux (34 / 10),
# grad_edge (16 / 36) and the diffusion edge flux (2 / 2) as gather.
AUTO_PFOLD_RATIO = 6


def auto_schedule(loop) -> str:
    """The INC schedule "auto" resolves to for ``loop`` (see AUTO_PFOLD_RATIO)."""
    if not fold_eligible(loop) or loop.iter_set.size == 0:
        return "gather"
    reads = sum(a.dat.dim for a in loop.args if a.kind == "indirect" and a.mode is READ)
    incs = [a for a in loop.args if a.kind == "indirect" and a.mode is INC]
    if reads < AUTO_PFOLD_RATIO * sum(a.dat.dim for a in incs):
        return "gather"
    return "pfold"


@dataclass
class BackendConfig:
    backend: str = "cuda"
    nthreads: int = 4                       # accepted for source compatibility; unused
    nranks: int = 1                         # GPUs (one process per GPU)
    block_size: int = 256
    block_size_table: dict | None = None    # per-loop block size overrides
    partitioner: str = "trivial"            # trivial | rcb (multi-GPU)
    coord_dat: str = "coords"
    balance: float = 1.0
    class_a_ranks: int = 1
    class_a_width: int = 4
    class_b_width: int = 1
    class_a_speed: float = 1.0
    class_b_speed: float = 1.0
    timeout_ms: float = 10000.0
    simulated_elem_cost: float = 0.0
    cost_model: Callable[[int], float] | None = None
    phase_callback: Callable[[str, int], None] | None = None
    # B200-specific
    device: int | None = None               # default: LOCAL_RANK or 0
    use_graph: bool = False                 # replay the program as one CUDA graph
    time_loops: bool = True                 # per-loop CUDA-event timing (eager mode)
    residency: str = "device"               # "device": lazy; "host": copy in/out every run
    inc_schedule: str = "auto"              # "auto" | "gather" | "pfold" | "colour"
    inc_schedule_table: dict | None = None  # per-loop override (tuner.tune_schedule)
    concurrent_loops: bool = True           # graphs/untimed runs: independent loops overlap on streams
    chain_loops: bool = True                # run registered adjacent loop pairs as one loop (chain.py)

    def __post_init__(self):
        if self.backend not in _BACKENDS:
            raise MeshError(f"unknown backend {self.backend!r}; expected one of {_BACKENDS} "
                            f"(the CPU backends live in the reference package)")
        if self.nthreads < 1 or self.nranks < 1 or self.block_size < 1:
            raise MeshError("nthreads, nranks and block_size must be positive")
        if self.balance <= 0:
            raise MeshError(f"balance must be positive, got {self.balance}")
        if self.partitioner not in ("trivial", "rcb"):
            raise MeshError(f"unknown partitioner {self.partitioner!r}")
        if self.residency not in ("device", "host"):
            raise MeshError(f"unknown residency {self.residency!r}")
        for sched in [self.inc_schedule, *(self.inc_schedule_table or {}).values()]:
            if sched not in SCHEDULES:
                raise MeshError(f"unknown inc_schedule {sched!r}; expected one of {SCHEDULES}")

    def schedule_for(self, loop_name: str) -> str:
        """The INC schedule of one loop ("pfold" falls back to "gather", "gather"
        to "colour" for loops they do not apply to)."""
        if self.inc_schedule_table and loop_name in self.inc_schedule_table:
            return self.inc_schedule_table[loop_name]
        return self.inc_schedule

    def block_size_for(self, loop_name: str) -> int:
        if self.block_size_table and loop_name in self.block_size_table:
            return int(self.block_size_table[loop_name])
        return self.block_size

    def device_index(self) -> int:
        if self.device is not None:
            return int(self.device)
        return int(os.environ.get("LOCAL_RANK", "0"))


@dataclass
class RunResult:
    perf: list[PerfRecord]
    total_sec: float
    messages: int = 0
    layout: object = None
    assignments: dict | None = None


def reduce_global(partials: Sequence, mode, initial=None):
    """Combine partials in the given order (reference executor.py:123-143)."""
    if mode not in (INC, MIN, MAX):
        raise MeshError(f"mode {mode} is not a reduction")
    arrs = [np.atleast_1d(np.asarray(p)) for p in partials]
    if initial is not None:
        acc = np.atleast_1d(np.asarray(initial)).copy()
    elif not arrs:
        raise MeshError("nothing to reduce")
    elif mode is INC:
        acc = np.zeros_like(arrs[0])
    else:
        acc, arrs = arrs[0].copy(), arrs[1:]
    op = {INC: np.add, MIN: np.minimum, MAX: np.maximum}[mode]
    for p in arrs:
        acc = op(acc, p)
    return acc[0] if acc.size == 1 else acc


# -- program compilation -------------------------------------------------------------

_KIND = {"direct": N.ML_DIRECT, "indirect": N.ML_INDIRECT, "global": N.ML_GLOBAL}


def _dtype_code(dt) -> int:
    return N.ML_F64 if np.dtype(dt) == np.float64 else N.ML_I64


def _functor_id(name: str, dtype: int, cache={}) -> int:
    key = (name, dtype)
    if key not in cache:
        fid = C.c_int32()
        N.check(N.lib().ml_functor_lookup(name.encode(), dtype, C.byref(fid)),
                f"kernel binding {name!r}")
        cache[key] = fid.value
    return cache[key]


def _functor_rec_cols(fid: int, cache={}) -> list | None:
    """Record column of each argument the functor declares (trait rec_cols), or None."""
    if fid not in cache:
        cols, n = (C.c_int8 * 64)(), C.c_int32()
        N.check(N.lib().ml_functor_rec_cols(fid, cols, C.byref(n)), "ml_functor_rec_cols")
        cache[fid] = list(cols[:n.value]) if n.value else None
    return cache[fid]


def _loop_dtype(loop: Loop) -> int:
    for a in loop.args:
        if a.kind != "global":
            return _dtype_code(a.dat.dtype)
    for a in loop.args:
        return _dtype_code(a.glob.dtype)
    return N.ML_F64


class _LoopEntry:
    """Everything one loop needs on the device, kept alive with the program."""

    def __init__(self, loop: Loop, mesh: Mesh, config: BackendConfig, gslot: dict,
                 garena_ptr: int, iter_counts: dict | None = None, rlim: dict | None = None):
        sname = loop.iter_set.name
        self.n = int(iter_counts[sname]) if iter_counts and sname in iter_counts else loop.iter_set.size
        self.loop = loop
        binding = resolve_kernel(loop.kernel)
        self.binding = binding
        self.functor = _functor_id(binding.functor, _loop_dtype(loop))
        self.bs = config.block_size_for(loop.name)
        self.plan = plan_for(loop, mesh, self.bs,
                             None if self.n == loop.iter_set.size else self.n)
        self.st = plan_stats(self.plan)
        pm = plan_mirror(self.plan)
        self.pm = pm
        args = (N.MlArg * max(len(loop.args), 1))()
        self.dats = []
        for i, a in enumerate(loop.args):
            r = args[i]
            r.kind = _KIND[a.kind]
            r.mode = N.MODE_CODE[a.mode.name]
            if a.kind == "global":
                r.dim = a.glob.dim
                r.dtype = _dtype_code(a.glob.dtype)
                r.data = garena_ptr + gslot[id(a.glob)]
                continue
            d = a.dat
            r.dim = d.dim
            r.dtype = _dtype_code(d.dtype)
            r.layout = N.ML_AOS if d.layout.name == "AOS" else N.ML_SOA
            r.set_size = d.set.size
            self.dats.append(d)
            m = dat_mirror(d)
            r.data = m.ptr or None
            r.pitch = m.pitch
            r.seg_shift = m.seg_shift
            if a.kind == "indirect":
                r.slot = a.slot
                r.map = map_mirror(a.map) or None
                r.map_from = a.map.from_set.size
        self.args = args
        L = N.MlLoop()
        self.name = loop.name.encode()
        L.name = self.name
        L.functor = self.functor
        L.nargs = len(loop.args)
        L.args = C.cast(args, C.POINTER(N.MlArg))
        L.n = self.n
        L.plan.nblocks = self.plan.nblocks
        L.plan.ncolors = self.plan.ncolors
        L.plan.block_size = self.bs
        L.plan.color_offsets = pm.offsets.ctypes.data_as(C.POINTER(C.c_int64))
        L.plan.blocks = pm.blocks.ptr
        L.plan.elem_color = pm.ecol.ptr if pm.ecol is not None else None
        L.plan.elem_ncolors = pm.encol.ptr if pm.encol is not None else None
        self.gather = None
        self.pfold = None
        self.pf_slots = None
        sched = config.schedule_for(loop.name)
        if sched == "auto":
            sched = auto_schedule(loop)
        if sched == "pfold" and not (self.n > 0 and fold_eligible(loop)):
            sched = "gather"
        self.sched = sched
        if sched == "pfold":
            self.gather = gather_mirror(loop, self.plan)
            pf = self.pfold = pfold_mirror(loop, self.plan)
            L.pf_n1, L.pf_off1, L.pf_elem1, L.pf_tl1 = pf.n1, pf.off1.ptr, pf.elem1.ptr, pf.tl1.ptr
            L.pf_n2, L.pf_off2, L.pf_elem2, L.pf_tl2 = pf.n2, pf.off2.ptr, pf.elem2.ptr, pf.tl2.ptr
            L.pf_pos2 = pf.pos2.ptr
            L.pf_slotpos = pf.slotpos.ptr
            L.pf_rec, L.pf_ncol = pf.rec.ptr, pf.ncol
            for w in (1, 2):
                if getattr(pf, f"seg{w}") is not None:
                    setattr(L, f"pf_seg{w}", getattr(pf, f"seg{w}").ptr)
                    setattr(L, f"pf_part{w}", getattr(pf, f"part{w}").ptr)
                    setattr(L, f"pf_nhub{w}", getattr(pf, f"nhub{w}"))
                    setattr(L, f"pf_hub{w}_tl", getattr(pf, f"hub{w}_tl").ptr)
                    setattr(L, f"pf_hub{w}_off", getattr(pf, f"hub{w}_off").ptr)
            for i, c in enumerate(pf.rcol):
                L.pf_rcol[i] = c
            L.functor = self.functor
            nb = C.c_uint64()
            N.check(N.lib().ml_loop_pfold_slot_bytes(C.byref(L), C.byref(nb)))
            self.pf_slots = N.DeviceBuffer(max(nb.value, 8))
            # slot rows are padded to whole 16-byte pairs that pass 2 copies in
            # full; zero the pads once (pass 1 never writes them)
            N.check(N.lib().ml_memset(self.pf_slots.ptr, 0, self.pf_slots.nbytes), "ml_memset")
            L.pf_slots = self.pf_slots.ptr
        elif sched == "gather" and self.n > 0 and gather_eligible(loop):
            self.gather = gather_mirror(loop, self.plan, hubs=True)
        if self.gather is not None and self.pfold is None:
            L.gather_ntargets = self.gather.ntargets
            L.gather_off = self.gather.off.ptr
            L.gather_elem = self.gather.elem.ptr
            L.gather_pos = self.gather.pos.ptr
            L.gather_targets = self.gather.targets.ptr if self.gather.targets is not None else None
            L.pf_rec, L.pf_ncol = self.gather.rec.ptr, self.gather.ncol
            for i, c in enumerate(self.gather.rcol):
                L.pf_rcol[i] = c
            if self.gather.seg is not None:
                g = self.gather
                L.gather_seg, L.gather_part, L.gather_nhub = g.seg.ptr, g.part.ptr, g.nhub
                L.gather_hub_tl, L.gather_hub_off = g.hub_tl.ptr, g.hub_off.ptr
        for k, v in enumerate(binding.fconsts[:4]):
            L.fconst[k] = v
        for k, v in enumerate(binding.iconsts[:4]):
            L.iconst[k] = v
        L.rlim = int(rlim[sname]) if rlim and sname in rlim else -1
        nbytes = C.c_uint64()
        N.check(N.lib().ml_loop_scratch_bytes(C.byref(L), C.byref(nbytes)))
        self.scratch = N.DeviceBuffer(nbytes.value) if nbytes.value else None
        if self.scratch:        # the last-CTA reduction ticket starts at zero
            N.check(N.lib().ml_memset(self.scratch.ptr, 0, nbytes.value), "ml_memset")
            N.check(N.lib().ml_synchronize(), "ml_synchronize")
        L.scratch = self.scratch.ptr if self.scratch else None
        # compile-time record columns (LP 2 kernels) when this loop's records
        # have exactly the columns the functor declares
        rcol = (self.pfold.rcol if self.pfold is not None else
                self.gather.rcol if self.gather is not None else None)
        want = _functor_rec_cols(self.functor) if rcol is not None else None
        if want is not None and len(want) == len(loop.args) and all(
                a.kind != "indirect" or rcol[i] == want[i] for i, a in enumerate(loop.args)):
            L.rec_fixed = 1
        self.desc = L
        self.useful = useful_bytes(loop)
        self.alg = b_alg(loop)
        self.written = [a.dat for a in loop.args if a.kind != "global" and a.mode in WRITE_MODES]

    def dat_pointers(self) -> tuple:
        return tuple(d._dev.ptr if d._dev is not None else 0 for d in self.dats)


class CompiledProgram:
    """A program bound to device state; replayable (optionally as a CUDA graph)."""

    def __init__(self, program: Sequence[Loop], mesh: Mesh, config: BackendConfig,
                 iter_counts: dict | None = None, rlim: dict | None = None):
        self.loops = list(program)
        # loops as launched: registered adjacent pairs fused (chain.py)
        # a loop a per-loop table names keeps its own entry: it is not fused
        pinned = frozenset(config.block_size_table or ()) | frozenset(config.inc_schedule_table or ())
        self.run_loops = chain_program(self.loops, mesh, pinned) if config.chain_loops else self.loops
        self.mesh = mesh
        self.version = mesh.version
        globs: list[Global] = []
        for loop in self.loops:
            for a in loop.args:
                if a.kind == "global" and all(g is not a.glob for g in globs):
                    globs.append(a.glob)
        self.globs = globs
        self.gslot, off = {}, 0
        for g in globs:
            self.gslot[id(g)] = off
            off += ((g.buffer.nbytes + 255) // 256) * 256
        self.gbytes = off
        self.gdev = N.DeviceBuffer(max(off, 256))
        self.ghost = N.PinnedArray((max(off, 256),), np.uint8)
        self.entries = [_LoopEntry(l, mesh, config, self.gslot, self.gdev.ptr, iter_counts, rlim)
                        for l in self.run_loops]
        self.all_dats = []
        for e in self.entries:
            for d in e.dats:
                if all(d is not x for x in self.all_dats):
                    self.all_dats.append(d)
        self.written = []
        for e in self.entries:
            for d in e.written:
                if all(d is not x for x in self.written):
                    self.written.append(d)
        descs = (N.MlLoop * max(len(self.entries), 1))(*[e.desc for e in self.entries])
        handle = C.c_void_p()
        N.check(N.lib().ml_program_create(descs, len(self.entries), self.ghost.array.ctypes.data,
                                          self.gdev.ptr, self.gbytes, C.byref(handle)),
                "ml_program_create")
        self.handle = handle.value
        N.check(N.lib().ml_program_set_concurrent(self.handle, int(bool(config.concurrent_loops))))
        self.ptrs = [e.dat_pointers() for e in self.entries]
        # each loop descriptor bakes its dats' layouts into strides (runtime.cu)
        self.layouts = [d.layout for d in self.all_dats]
        self.runs = 0

    def dependencies(self) -> list:
        """Per loop: (earlier loops it must wait for, stream lane) of the
        concurrent schedule (ml_program_deps)."""
        out = []
        for i in range(len(self.entries)):
            nd, lane = C.c_int32(), C.c_int32()
            N.check(N.lib().ml_program_deps(self.handle, i, C.byref(nd), None, C.byref(lane)))
            deps = (C.c_int32 * max(nd.value, 1))()
            N.check(N.lib().ml_program_deps(self.handle, i, C.byref(nd), deps, C.byref(lane)))
            out.append((list(deps[:nd.value]), lane.value))
        return out

    def valid_for(self, mesh: Mesh) -> bool:
        if mesh.version != self.version:
            return False
        if [d.layout for d in self.all_dats] != self.layouts:
            return False
        for d in self.all_dats:
            dat_mirror(d)
        return [e.dat_pointers() for e in self.entries] == self.ptrs

    def run(self, use_graph: bool, time_loops: bool, force_upload: bool = False):
        for d in self.all_dats:
            dat_mirror(d, force_upload=force_upload)
        hv = self.ghost.array
        for g in self.globs:
            o = self.gslot[id(g)]
            hv[o:o + g.buffer.nbytes] = g.buffer.view(np.uint8)
        timed = bool(time_loops) and not use_graph
        N.check(N.lib().ml_program_run(self.handle, int(bool(use_graph)), int(timed)),
                f"program [{', '.join(l.name for l in self.loops[:4])}...]")
        for g in self.globs:
            o = self.gslot[id(g)]
            g.buffer[:] = hv[o:o + g.buffer.nbytes].view(g.buffer.dtype)
        for d in self.written:
            d._dev.device_newer = True
        self.runs += 1
        if timed:
            ms = (C.c_float * max(len(self.entries), 1))()
            N.check(N.lib().ml_program_loop_times(self.handle, ms))
            return [float(ms[i]) * 1e-3 for i in range(len(self.entries))]
        return None

    def run_phases(self, callback) -> None:
        """Eager run with the reference's per-phase hook (executor.py:251-252):
        a loop on the colour schedule is launched one block colour at a time,
        ``callback(loop name, colour)`` called before each colour, with the
        device synchronised after it; loops on the target-centric and direct
        schedules have no colour phases and run without callbacks."""
        L = N.lib()
        for d in self.all_dats:
            dat_mirror(d)
        hv = self.ghost.array
        for g in self.globs:
            o = self.gslot[id(g)]
            hv[o:o + g.buffer.nbytes] = g.buffer.view(np.uint8)
        N.check(L.ml_upload(self.gdev.ptr, N.ptr(hv), self.gbytes), "ml_upload")
        for e in self.entries:
            coloured = (e.gather is None and e.pfold is None and e.plan.has_writes and e.n > 0)
            if not coloured:
                N.check(L.ml_loop_run(C.byref(e.desc)), f"loop {e.loop.name!r}")
                continue
            for c in range(e.plan.ncolors):
                callback(e.loop.name, c)
                desc = type(e.desc).from_buffer_copy(e.desc)
                desc.colour_begin, desc.colour_end = c, c + 1
                N.check(L.ml_loop_run(C.byref(desc)), f"loop {e.loop.name!r} colour {c}")
                N.check(L.ml_synchronize(), "ml_synchronize")
        N.check(L.ml_download(N.ptr(hv), self.gdev.ptr, self.gbytes), "ml_download")
        for g in self.globs:
            o = self.gslot[id(g)]
            g.buffer[:] = hv[o:o + g.buffer.nbytes].view(g.buffer.dtype)
        for d in self.written:
            d._dev.device_newer = True
        self.runs += 1

    def _stream_plan(self):
        """Per loop: the input dats first used there (uploaded just before it)
        and the written dats last written there (downloaded right after it).
        A dat is an input unless its first access overwrites the whole set
        (a direct WRITE over the full iteration set, not also read there)."""
        plan = self.__dict__.get("_splan")
        if plan is not None:
            return plan
        first, last = [[] for _ in self.entries], [[] for _ in self.entries]
        seen, last_w = set(), {}
        for i, e in enumerate(self.entries):
            loop = e.loop
            for d in e.dats:
                key = id(d)
                if key in seen:
                    continue
                seen.add(key)
                modes = [a for a in loop.args if a.kind != "global" and a.dat is d]
                overwrite = (all(a.kind == "direct" and a.mode.name == "WRITE" for a in modes)
                             and e.n == d.set.size)
                if not overwrite:
                    first[i].append(d)
            for d in e.written:
                last_w[id(d)] = (i, d)
        for i, d in last_w.values():
            last[i].append(d)
        self._splan = (first, last)
        return self._splan

    def run_streamed(self) -> None:
        """Host-resident run with the copies overlapped with execution: each
        input dat is uploaded (H2D stream) just before the first loop that uses
        it, each written dat downloaded (D2H stream) right after its last
        writer, while the compute stream runs the loops (stream-ordered with
        events, one host synchronisation at the end)."""
        L = N.lib()
        first, last = self._stream_plan()
        hv = self.ghost.array
        for g in self.globs:
            o = self.gslot[id(g)]
            hv[o:o + g.buffer.nbytes] = g.buffer.view(np.uint8)
        # a dat whose device copy is newer than the host payload (left by a
        # device-resident run) is already current on the device: uploading the
        # stale host copy would lose it
        stale_host = {id(d) for d in self.all_dats if d._dev is not None and d._dev.device_newer}
        for d in self.all_dats:
            dat_mirror(d, upload=False)        # allocation; contents come below
        N.check(L.ml_copy_h2d(self.gdev.ptr, N.ptr(hv), self.gbytes), "ml_copy_h2d")
        uploaded = []
        for i, e in enumerate(self.entries):
            for d in first[i]:
                if id(d) in stale_host:
                    continue
                uploaded.append(d)
                host = d._host
                if host.nbytes:
                    if not host.flags.c_contiguous:
                        d._host = host = np.ascontiguousarray(host)
                    d._dev.copy_h2d(host)
            if first[i] or i == 0:
                N.check(L.ml_order(N.ML_STREAM_H2D, N.ML_STREAM_COMPUTE))
            N.check(L.ml_loop_run(C.byref(e.desc)), f"loop {e.loop.name!r}")
            if last[i]:
                N.check(L.ml_order(N.ML_STREAM_COMPUTE, N.ML_STREAM_D2H))
                for d in last[i]:
                    d._dev.copy_d2h(d._host)
        N.check(L.ml_order(N.ML_STREAM_COMPUTE, N.ML_STREAM_D2H))
        N.check(L.ml_copy_d2h(N.ptr(hv), self.gdev.ptr, self.gbytes), "ml_copy_d2h")
        N.check(L.ml_sync_all(), "ml_sync_all")
        for g in self.globs:
            o = self.gslot[id(g)]
            g.buffer[:] = hv[o:o + g.buffer.nbytes].view(g.buffer.dtype)
        for d in uploaded:
            d._dev.host_newer = False
        for d in self.written:                 # downloaded after their last writer
            d._dev.host_newer = False
            d._dev.device_newer = False
        self.runs += 1

    def replay(self, count: int) -> None:
        """``count`` back-to-back CUDA-graph replays (device throughput; globals
        are written back to the host once, after the last replay)."""
        for d in self.all_dats:
            dat_mirror(d)
        hv = self.ghost.array
        for g in self.globs:
            o = self.gslot[id(g)]
            hv[o:o + g.buffer.nbytes] = g.buffer.view(np.uint8)
        N.check(N.lib().ml_program_replay(self.handle, int(count)), "ml_program_replay")
        for g in self.globs:
            o = self.gslot[id(g)]
            g.buffer[:] = hv[o:o + g.buffer.nbytes].view(g.buffer.dtype)
        for d in self.written:
            d._dev.device_newer = True
        self.runs += count

    def replay_timed(self, count: int) -> list:
        """Per-loop device seconds of the steady-state CUDA graph (mean of
        ``count`` replays of a sequential capture with timing events between
        loops); globals are written back as after a run."""
        for d in self.all_dats:
            dat_mirror(d)
        hv = self.ghost.array
        for g in self.globs:
            o = self.gslot[id(g)]
            hv[o:o + g.buffer.nbytes] = g.buffer.view(np.uint8)
        ms = (C.c_float * max(len(self.entries), 1))()
        N.check(N.lib().ml_program_replay_timed(self.handle, int(count), ms), "ml_program_replay_timed")
        for g in self.globs:
            o = self.gslot[id(g)]
            g.buffer[:] = hv[o:o + g.buffer.nbytes].view(g.buffer.dtype)
        for d in self.written:
            d._dev.device_newer = True
        self.runs += count
        return [float(ms[i]) * 1e-3 for i in range(len(self.entries))]

    def launches_per_run(self) -> int:
        """Kernel launches one run enqueues (colour launches + reduction combines)."""
        total = 0
        for e in self.entries:
            if e.loop.iter_set.size == 0:
                continue
            if e.pfold is not None:
                total += 1 + (1 if e.pfold.n2 > 0 else 0) + (1 if e.pfold.nhub1 else 0) + (
                    1 if e.pfold.n2 > 0 and e.pfold.nhub2 else 0)
            elif e.gather is not None or not e.plan.has_writes:
                total += 1 + (1 if e.gather is not None and e.gather.nhub else 0)
            else:
                total += e.plan.ncolors
                # colour schedules fold reduction partials with k_combine; the
                # single-launch schedules fold them in their last CTA
                total += sum(1 for a in e.loop.args if a.kind == "global" and a.mode.name != "READ")
        return total

    def __del__(self):
        h = getattr(self, "handle", None)
        if h and N._lib is not None:
            N._lib.ml_program_free(h)
            self.handle = None


_PROGRAM_CACHE_SIZE = 32


def compile_program(program: Sequence[Loop], mesh: Mesh, config: BackendConfig,
                    iter_counts: dict | None = None, rlim: dict | None = None) -> CompiledProgram:
    """Compiled program for (loops, block sizes, mesh version), cached on the mesh.

    ``iter_counts`` (set name -> n) runs loops over a prefix of their iteration
    set and ``rlim`` (set name -> n) limits global reductions to a prefix —
    the owned / owned+exec-halo split of a multi-GPU rank."""
    N.init(config.device_index())
    cache = mesh.__dict__.setdefault("_ml_programs", OrderedDict())
    key = (tuple(id(l) for l in program),
           tuple(config.block_size_for(l.name) for l in program), config.block_size,
           tuple(sorted((config.block_size_table or {}).items())), config.inc_schedule,
           tuple(sorted((config.inc_schedule_table or {}).items())), config.coord_dat,
           config.concurrent_loops, config.chain_loops,
           tuple(sorted((iter_counts or {}).items())), tuple(sorted((rlim or {}).items())))
    cp = cache.get(key)
    if cp is not None and cp.loops == list(program) and cp.valid_for(mesh):
        cache.move_to_end(key)
        return cp
    cp = CompiledProgram(program, mesh, config, iter_counts, rlim)
    cache[key] = cp
    while len(cache) > _PROGRAM_CACHE_SIZE:
        cache.popitem(last=False)
    return cp


def _sync_host(dats) -> None:
    for d in dats:
        d._pull()


def _record(collector: PerfCollector, cp: CompiledProgram, times) -> None:
    for e, t in zip(cp.entries, times):
        collector.add(e.loop.name, t, e.useful, nb=e.st.nb, nc=e.st.nc, alg_bytes=e.alg)


def run_program(program: Sequence[Loop], mesh: Mesh, config: BackendConfig | None = None
                ) -> RunResult:
    """Execute a loop program on B200 and collect per-loop device timings.

    ``mesh`` may also be a reference ``meshloop.Mesh`` with a program of
    reference objects (run through :mod:`.foreign`: shadow mesh sharing its
    arrays, host-resident coherence)."""
    if not isinstance(mesh, Mesh):
        from .foreign import run_foreign
        return run_foreign(program, mesh, config)
    config = config or BackendConfig()
    world = int(os.environ.get("WORLD_SIZE", "1"))
    if config.nranks > 1 or world > 1:
        from .multigpu import run_program_distributed
        return run_program_distributed(program, mesh, config)
    mesh.freeze()
    t0 = time.perf_counter()
    collector = PerfCollector()
    program = list(program)
    if not program:
        return RunResult([], 0.0)
    cp = compile_program(program, mesh, config)
    if config.phase_callback is not None:
        cp.run_phases(config.phase_callback)
        if config.residency == "host":
            _sync_host(cp.written)
        return RunResult(collector.finalize(), time.perf_counter() - t0)
    host = config.residency == "host"
    if host and (config.use_graph or not config.time_loops):
        cp.run_streamed()
        times = None
    else:
        times = cp.run(config.use_graph, config.time_loops, force_upload=host)
        if host:
            _sync_host(cp.written)
    if times is not None:
        _record(collector, cp, times)
    return RunResult(collector.finalize(), time.perf_counter() - t0)


def run_loop(loop: Loop, mesh: Mesh, config: BackendConfig | None = None,
             collector: PerfCollector | None = None) -> None:
    """Execute one loop (the per-loop entry of reference executor.py:206/278)."""
    config = config or BackendConfig()
    mesh.freeze()
    cp = compile_program([loop], mesh, config)
    if config.phase_callback is not None:
        cp.run_phases(config.phase_callback)
        return
    times = cp.run(False, config.time_loops or collector is not None)
    if collector is not None and times is not None:
        _record(collector, cp, times)


def run_serial(loop: Loop, mesh: Mesh, config: BackendConfig | None = None,
               collector: PerfCollector | None = None) -> None:
    """Reference ``run_serial`` (executor.py:206-217) on the device: indirect
    increments use the target-centric schedule, which applies every target's
    increments in ascending element order — the serial result, bit for bit.
    Loops with indirect WRITE/RW arguments run coloured (as the reference's
    parallel backends do)."""
    from dataclasses import replace
    run_loop(loop, mesh, replace(config or BackendConfig(), inc_schedule="gather"), collector)


def run_threads(loop: Loop, mesh: Mesh, config: BackendConfig | None = None,
                collector: PerfCollector | None = None) -> None:
    """Reference ``run_threads`` (executor.py:278-284): the coloured schedule of
    the reference plan (block colours in order, element colours inside a block)
    as per-colour CUDA launches."""
    from dataclasses import replace
    run_loop(loop, mesh, replace(config or BackendConfig(), inc_schedule="colour"), collector)


def run_ranks(program: Sequence[Loop], mesh: Mesh, layout=None,
              config: BackendConfig | None = None,
              collector: PerfCollector | None = None) -> RunResult:
    """Reference ``run_ranks`` (executor.py:690-695): owner-compute execution over
    ``layout`` (or the layout of ``config``), one process per GPU — launch with
    torchrun; the ranks are processes, not threads of this one."""
    from .multigpu import run_program_distributed
    config = config or BackendConfig(nranks=layout.nranks if layout is not None else 1)
    return run_program_distributed(program, mesh, config, layout=layout, collector=collector)


def run_hybrid(program: Sequence[Loop], mesh: Mesh, config: BackendConfig | None = None,
               collector: PerfCollector | None = None) -> RunResult:
    """Reference ``run_hybrid`` (executor.py:698-704) mixes CPU worker classes; on
    B200 there is no CPU execution path, so this is refused loudly."""
    raise ExecError("run_hybrid: CPU+GPU hybrid execution is not provided by the B200 backend; "
                    "use run_program (one GPU) or run_ranks (one process per GPU)")
