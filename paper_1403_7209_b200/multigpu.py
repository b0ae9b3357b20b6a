"""Owner-compute multi-GPU execution: one process per GPU.

Semantic model: the reference ranks backend (executor.py:300-329 layout,
367-574 rank context, 577-600 rank main loop, 603-627 dat roles, 630-687
program driver).  Each rank:

1. builds the same layout as the reference (``build_layout``: partition the
   map target sets — trivial or RCB — derive iteration-set ownership, close
   exec / non-exec halos; bit-exact with the reference, golden-tested);
2. builds a *local mesh* numbered ``[owned | exec halo | non-exec halo]``
   (reference ``SetHalos.local_ids``) holding only what its elements touch;
3. executes, per program entry, the owned + exec-halo elements of the
   iteration set on its GPU; global reductions only count the owned prefix
   (``rlim``, reference executor.py:519-524);
4. exchanges a dat's halo lazily — before a loop that reads it after some
   loop wrote it (reference dirty bits, executor.py:582-595) — by packing the
   export rows on the device, moving them with the transport, and scattering
   them into the import slots;
5. after every reducing loop, gathers the per-rank partials and folds them
   in ascending rank order onto the running value (so a MIN computed by one
   loop is the value a later loop READs, as in serial execution — the
   reference's ranks backend instead exposes the initial value until the
   program ends);
6. at the end, all-gathers owned rows so every rank's dats and globals hold
   the full result.

Transports: ``"nccl"`` (torch.distributed NCCL on device buffers, ordered on
the library's stream; the production path on 2-8 B200s) and ``"gloo"``
(host-staged; used to test the protocol with several ranks on one GPU and,
with an injected CPU executor, on CPU).
"""
from __future__ import annotations

import os
from collections import OrderedDict
import time
from dataclasses import dataclass, field
from typing import Sequence

import numpy as np

from .core import (INC, MAX, MIN, READ, RW, SOA, WRITE_MODES, ExecError, Global, Loop, Mesh,
                   MeshError, arg_direct, arg_global, arg_indirect, transform_layout)
from .partition import (RankLayout, build_halos, derive_assignments, partition_rcb,
                        partition_trivial)

__all__ = ["build_layout", "RankProgram", "run_program_distributed", "bench_distributed",
           "unique_loops", "loop_dat_roles"]


def unique_loops(program: Sequence[Loop]) -> list[Loop]:
    seen, out = set(), []
    for loop in program:
        sig = loop.signature()
        if sig not in seen:
            seen.add(sig)
            out.append(loop)
    return out


def build_layout(mesh: Mesh, program: Sequence[Loop], config) -> RankLayout:
    """Partition every touched set and close the halos (reference executor.py:300-329)."""
    loops = unique_loops(program)
    targets = []
    for loop in loops:
        for a in loop.args:
            if a.kind == "indirect" and a.map.to_set not in targets:
                targets.append(a.map.to_set)
    base = {}
    for s in targets:
        if config.partitioner == "rcb":
            coords = mesh.dats.get(config.coord_dat)
            if coords is None or coords.set is not s:
                raise MeshError(f"rcb partitioning needs coordinates dat {config.coord_dat!r} "
                                f"on set {s.name!r}")
            base[s.name] = partition_rcb(coords, config.nranks)
        else:
            base[s.name] = partition_trivial(s, config.nranks)
    return build_halos(mesh, loops, derive_assignments(mesh, loops, base, config.nranks))


def loop_dat_roles(program: Sequence[Loop], layout: RankLayout):
    """Per program entry: dats needing fresh halos before, dats written after
    (reference executor.py:603-627)."""
    roles = []
    for loop in program:
        redundant = any(layout.sets[loop.iter_set.name][r].exec_halo.size
                        for r in range(layout.nranks))
        reads, writes = [], []
        for a in loop.args:
            if a.dat is None:
                continue
            if (a.mode in (READ, RW) and (a.kind == "indirect" or redundant)
                    and a.dat.name not in reads):
                reads.append(a.dat.name)
            if a.mode in WRITE_MODES and a.dat.name not in writes:
                writes.append(a.dat.name)
        roles.append((reads, writes))
    return roles


def _identity(mode, dtype, dim):
    dtype = np.dtype(dtype)
    if mode is INC:
        return np.zeros(dim, dtype)
    if dtype.kind == "i":
        return np.full(dim, np.iinfo(dtype).max if mode is MIN else np.iinfo(dtype).min, dtype)
    return np.full(dim, np.inf if mode is MIN else -np.inf, dtype)


def fold(value: np.ndarray, partials, mode) -> np.ndarray:
    """value ⊕ p_0 ⊕ p_1 ⊕ ... in the given (rank) order."""
    op = {INC: np.add, MIN: np.minimum, MAX: np.maximum}[mode]
    out = np.array(value, copy=True)
    for p in partials:
        out = op(out, p)
    return out


@dataclass
class Exchange:
    """Export / import local ids of one set on one rank."""
    exports: dict = field(default_factory=dict)      # dst -> local ids (int32)
    imports: dict = field(default_factory=dict)      # src -> local ids (int32)


class RankProgram:
    """One rank's slice of a program: local mesh, loops, counts and exchange lists."""

    def __init__(self, mesh: Mesh, program: Sequence[Loop], layout: RankLayout, rank: int):
        self.rank, self.nranks = rank, layout.nranks
        self.layout = layout
        self.program = list(program)
        self.local = Mesh(auto_soa_threshold=None)
        self.local_ids: dict[str, np.ndarray] = {}
        self.g2l: dict[str, np.ndarray] = {}
        self.n_exec: dict[str, int] = {}
        self.n_owned: dict[str, int] = {}
        self.exchange: dict[str, Exchange] = {}
        sets = {}
        for name in mesh.sets:                                   # global declaration order
            if name not in layout.sets:
                continue
            h = layout.sets[name][rank]
            ids = h.local_ids.astype(np.int64)
            g2l = np.full(mesh.sets[name].size, -1, np.int64)
            g2l[ids] = np.arange(ids.size)
            self.local_ids[name], self.g2l[name] = ids, g2l
            self.n_owned[name] = int(h.owned.size)
            self.n_exec[name] = int(h.owned.size + h.exec_halo.size)
            sets[name] = self.local.decl_set(name, int(ids.size))
            self.exchange[name] = Exchange(
                {d: g2l[v].astype(np.int32) for d, v in sorted(h.exports.items())},
                {s: g2l[v].astype(np.int32) for s, v in sorted(h.imports.items())})
        maps = {}
        for loop in self.program:
            for a in loop.args:
                if a.kind != "indirect" or a.map.name in maps:
                    continue
                m = a.map
                rows = self.local_ids[m.from_set.name]
                t = self.g2l[m.to_set.name][m.table[rows]]
                ne = self.n_exec[m.from_set.name]
                if (t[:ne] < 0).any():
                    raise ExecError(f"rank {rank}: map {m.name!r} leaves the halo closure")
                t[ne:][t[ne:] < 0] = 0          # rows of never-executed halo elements
                maps[m.name] = self.local.decl_map(m.name, sets[m.from_set.name],
                                                   sets[m.to_set.name], m.arity, (t + 1).ravel())
        dats = {}
        for loop in self.program:
            for a in loop.args:
                if a.dat is None or a.dat.name in dats:
                    continue
                d = a.dat
                vals = d.fetch()[self.local_ids[d.set.name]]
                ld = self.local.decl_dat(d.name, sets[d.set.name], d.dim, d.dtype.name, vals.ravel())
                if d.layout is SOA:
                    transform_layout(ld, SOA)
                dats[d.name] = ld
        self.global_dats = {name: mesh.dats[name] for name in dats}
        self.dats = dats
        # globals: one running value per global; one identity partial per reducing arg
        self.values: dict[int, Global] = {}
        self.partials: dict[tuple, Global] = {}
        self.user_globals: dict[int, Global] = {}
        self.loops: list[Loop] = []
        self.reductions: list[list] = []          # per entry: [(partial Global, value Global, mode)]
        for i, loop in enumerate(self.program):
            args, reds = [], []
            for j, a in enumerate(loop.args):
                if a.kind == "global":
                    g = a.glob
                    self.user_globals[id(g)] = g
                    val = self.values.setdefault(id(g), Global(g.buffer.copy(), name=g.name))
                    if a.mode is READ:
                        args.append(arg_global(val, READ))
                    else:
                        part = Global(_identity(a.mode, g.dtype, g.dim), name=f"{g.name}@{i}.{j}")
                        self.partials[(i, j)] = part
                        reds.append((part, val, a.mode))
                        args.append(arg_global(part, a.mode))
                elif a.kind == "direct":
                    args.append(arg_direct(dats[a.dat.name], a.mode))
                else:
                    args.append(arg_indirect(dats[a.dat.name], maps[a.map.name], a.slot + 1, a.mode))
            self.loops.append(Loop(loop.name, sets[loop.iter_set.name], args, loop.kernel))
            self.reductions.append(reds)
        self.roles = loop_dat_roles(self.program, layout)

    def refresh_from_global(self) -> None:
        """Re-read every local dat (owned + halo rows) from the global mesh — the
        user-visible truth between runs — and mark all halos fresh."""
        for name, ld in self.dats.items():
            gd = self.global_dats[name]
            ld.put(gd.fetch()[self.local_ids[gd.set.name]])
        self.__dict__["dirty"] = {}
        self.refresh_globals()

    def reset_partials(self, entry: int) -> None:
        for part, _val, mode in self.reductions[entry]:
            part.buffer[:] = _identity(mode, part.dtype, part.dim)

    def refresh_globals(self) -> None:
        """Re-read user global values (a new run starts from the user's buffers)."""
        for gid, val in self.values.items():
            val.buffer[:] = self.user_globals[gid].buffer

    def halo_rows(self, dat_name: str) -> tuple[dict, dict]:
        ex = self.exchange[self.dats[dat_name].set.name]
        return ex.exports, ex.imports

    def owned_rows(self, dat_name: str) -> np.ndarray:
        d = self.dats[dat_name]
        return d.fetch()[: self.n_owned[d.set.name]]


# -- transports ------------------------------------------------------------------------------

class GlooTransport:
    """Host-staged point-to-point and all-gather over torch.distributed (gloo)."""

    name = "gloo"

    def __init__(self, group=None):
        import torch
        import torch.distributed as dist
        self.torch, self.dist, self.group = torch, dist, group

    def exchange(self, sends: dict, recv_shapes: dict, dtype) -> dict:
        torch, dist = self.torch, self.dist
        ops, bufs = [], {}
        for dst, arr in sorted(sends.items()):
            ops.append(dist.P2POp(dist.isend, torch.from_numpy(np.ascontiguousarray(arr)), dst,
                                  group=self.group))
        for src, shape in sorted(recv_shapes.items()):
            bufs[src] = torch.empty(shape, dtype=torch.float64 if np.dtype(dtype) == np.float64
                                    else torch.int64)
            ops.append(dist.P2POp(dist.irecv, bufs[src], src, group=self.group))
        if ops:
            for req in dist.batch_isend_irecv(ops):
                req.wait()
        return {s: b.numpy() for s, b in bufs.items()}

    def allgather(self, arr: np.ndarray) -> list:
        torch, dist = self.torch, self.dist
        t = torch.from_numpy(np.ascontiguousarray(arr))
        out = [torch.empty_like(t) for _ in range(dist.get_world_size(self.group))]
        dist.all_gather(out, t, group=self.group)
        return [o.numpy() for o in out]

    def allgather_object(self, obj) -> list:
        out = [None] * self.dist.get_world_size(self.group)
        self.dist.all_gather_object(out, obj, group=self.group)
        return out

    def barrier(self):
        self.dist.barrier(group=self.group)

    # device collectives used by StreamRank (host-staged for gloo)
    def sendrecv_device(self, sends: dict, recvs: dict, stream) -> None:
        from . import _native as N
        N.check(N.lib().ml_synchronize(), "ml_synchronize")
        got = self.exchange({d: t.cpu().numpy() for d, t in sends.items()},
                            {s: tuple(t.shape) for s, t in recvs.items()}, np.float64 if all(
                                t.dtype == self.torch.float64 for t in recvs.values()) else np.int64)
        with self.torch.cuda.stream(stream):
            for src, t in recvs.items():
                t.copy_(self.torch.from_numpy(got[src]).to(t.device))
        stream.synchronize()

    def allgather_device(self, out, inp, stream) -> None:
        from . import _native as N
        N.check(N.lib().ml_synchronize(), "ml_synchronize")
        parts = self.allgather(inp.cpu().numpy())
        with self.torch.cuda.stream(stream):
            out.copy_(self.torch.from_numpy(np.concatenate(parts)).to(out.device))
        stream.synchronize()

    # device-buffer interface (DeviceRank): device staging + pinned host mirror
    def buffer(self, key, n: int, dtype):
        from . import _native as N
        cache = self.__dict__.setdefault("_bufs", {})
        if key not in cache or cache[key][0].nbytes < max(8 * n, 8):
            cache[key] = (N.DeviceBuffer(max(8 * n, 8)), N.PinnedArray((max(n, 1),), dtype), n)
        return cache[key]

    @staticmethod
    def ptr(buf) -> int:
        return buf[0].ptr

    def sendrecv(self, sends: dict, recvs: dict, dtype) -> None:
        from . import _native as N
        L = N.lib()
        for dev, host, n in sends.values():
            N.check(L.ml_download(N.ptr(host.array), dev.ptr, 8 * n), "ml_download")
        got = self.exchange({d: b[1].array[:b[2]] for d, b in sends.items()},
                            {s: (b[2],) for s, b in recvs.items()}, dtype)
        for src, (dev, host, n) in recvs.items():
            host.array[:n] = got[src]
            N.check(L.ml_upload(dev.ptr, N.ptr(host.array), 8 * n), "ml_upload")


class NcclTransport(GlooTransport):
    """Device-to-device halo exchange with torch.distributed's NCCL backend.

    Send/receive buffers are CUDA tensors; ``ml_pack_rows`` writes into them
    on the library stream, which is synchronised before the grouped NCCL
    send/recv (batch_isend_irecv) and the receive side is synchronised before
    ``ml_unpack_rows`` scatters the rows into the import slots."""

    name = "nccl"

    def buffer(self, key, n: int, dtype):
        cache = self.__dict__.setdefault("_bufs", {})
        torch = self.torch
        if key not in cache or cache[key].numel() < max(n, 1):
            tdt = torch.float64 if np.dtype(dtype) == np.float64 else torch.int64
            cache[key] = torch.empty(max(n, 1), dtype=tdt, device="cuda")
        return cache[key][:max(n, 1)] if n else cache[key][:0]

    @staticmethod
    def ptr(buf) -> int:
        return buf.data_ptr()

    def sendrecv(self, sends: dict, recvs: dict, dtype=None) -> None:
        from . import _native as N
        N.check(N.lib().ml_synchronize(), "ml_synchronize")
        dist = self.dist
        ops = [dist.P2POp(dist.isend, t, dst, group=self.group) for dst, t in sorted(sends.items())]
        ops += [dist.P2POp(dist.irecv, t, src, group=self.group) for src, t in sorted(recvs.items())]
        if ops:
            for req in dist.batch_isend_irecv(ops):
                req.wait()
        self.torch.cuda.current_stream().synchronize()

    def exchange(self, sends: dict, recv_shapes: dict, dtype) -> dict:
        raise ExecError("NcclTransport moves device buffers only")

    # stream-ordered device collectives (StreamRank): issued with `stream` current,
    # so NCCL waits for the packing kernels and the stream waits for NCCL
    def sendrecv_stream(self, sends: dict, recvs: dict) -> None:
        dist = self.dist
        ops = [dist.P2POp(dist.isend, t, dst, group=self.group) for dst, t in sorted(sends.items())]
        ops += [dist.P2POp(dist.irecv, t, src, group=self.group) for src, t in sorted(recvs.items())]
        if ops:
            for w in dist.batch_isend_irecv(ops):
                w.wait()

    def sendrecv_device(self, sends: dict, recvs: dict, stream) -> None:
        with self.torch.cuda.stream(stream):
            self.sendrecv_stream(sends, recvs)

    def allgather_device(self, out, inp, stream) -> None:
        with self.torch.cuda.stream(stream):
            self.dist.all_gather_into_tensor(out, inp, group=self.group)

    def allgather(self, arr: np.ndarray) -> list:
        torch = self.torch
        t = torch.from_numpy(np.ascontiguousarray(arr)).cuda()
        out = [torch.empty_like(t) for _ in range(self.dist.get_world_size(self.group))]
        self.dist.all_gather(out, t, group=self.group)
        return [o.cpu().numpy() for o in out]


# -- device execution ------------------------------------------------------------------------

class DeviceRank:
    """Runs a RankProgram's loops on this rank's GPU through libmeshloop_b200."""

    def __init__(self, rp: RankProgram, config):
        from .executor import compile_program
        self.rp, self.config = rp, config
        self.progs = [compile_program([l], rp.local, config, iter_counts=rp.n_exec,
                                      rlim=rp.n_owned) for l in rp.loops]

    def run_loop(self, i: int, use_graph: bool = False) -> float:
        self.rp.reset_partials(i)
        t = self.progs[i].run(use_graph, not use_graph)
        return t[0] if t else 0.0

    # halo exchange on the device: pack export rows (ml_pack_rows), move them,
    # scatter into import slots (ml_unpack_rows); reference executor.py:484-497
    def _index(self, key, ids: np.ndarray):
        from . import _native as N
        cache = self.__dict__.setdefault("_idx", {})
        if key not in cache:
            buf = N.DeviceBuffer(max(ids.nbytes, 4))
            if ids.size:
                buf.upload(np.ascontiguousarray(ids, dtype=np.int32))
            cache[key] = buf
        return cache[key]

    def exchange_halo(self, name: str, transport) -> int:
        from . import _native as N
        from .device import dat_mirror
        d = self.rp.dats[name]
        m = dat_mirror(d)
        se, sc = m.strides(d)
        exports, imports = self.rp.halo_rows(name)
        L = N.lib()
        sends = {}
        for dst, ids in exports.items():
            buf = transport.buffer(("s", name, dst), ids.size * d.dim, d.dtype)
            N.check(L.ml_pack_rows(transport.ptr(buf), m.ptr, self._index(("e", name, dst), ids).ptr,
                                   ids.size, d.dim, se, sc), "ml_pack_rows")
            sends[dst] = buf
        recvs = {src: transport.buffer(("r", name, src), ids.size * d.dim, d.dtype)
                 for src, ids in imports.items()}
        transport.sendrecv(sends, recvs, d.dtype)
        for src, ids in imports.items():
            N.check(L.ml_unpack_rows(m.ptr, transport.ptr(recvs[src]),
                                     self._index(("i", name, src), ids).ptr, ids.size, d.dim, se, sc),
                    "ml_unpack_rows")
        m.device_newer = True
        return len(sends)


_LAST_HALO_PATH = ""
_LAST_OVERLAPPED: list = []          # (loop, schedule) split into core/boundary launches in the last run


class NvlinkHalo:
    """Halo exchange by direct peer stores (CUDA IPC over NVLink/NVSwitch).

    Each rank allocates, per (dat, source rank), the import buffer that source
    writes into, plus one arrival counter per source; handles are exchanged
    once (all-gather).  An exchange is then, on the compute stream: for every
    destination one ``ml_put_rows`` kernel that gathers the export rows
    straight into the destination's import buffer and bumps its arrival
    counter after a system-scope fence; for every source one ``ml_wait_flag``
    (device spin on the counter), the ``ml_unpack_rows`` scatter and a credit
    back to the source (``ml_signal_flag``): a producer puts only after the
    destination has consumed its previous delivery, so ranks may drift apart
    without overwriting an unread import buffer.  No host involvement and no
    NCCL on the halo path, so it is graph-capturable; the put overlaps
    whatever the stream runs before the wait (core targets)."""

    def __init__(self, rp: RankProgram, transport, timeout_ms: float = 10000.0):
        import ctypes as C
        from . import _native as N
        self.C, self.N, self.rp = C, N, rp
        self.timeout_ns = int(max(timeout_ms, 0.0) * 1e6)
        L = N.lib()
        self.local, self.remote, self.handles = {}, {}, {}
        self.opened = []
        nr = rp.nranks
        names = sorted({n for reads, _w in rp.roles for n in reads if n in rp.dats})
        keys = []
        for name in names:
            d = rp.dats[name]
            _ex, imports = rp.halo_rows(name)
            for src, ids in sorted(imports.items()):
                buf = N.DeviceBuffer(max(ids.size * d.dim * 8, 8))
                self.local[(name, src)] = buf
                keys.append((name, src))
        # per (dat, peer) counters: deliveries [ni*nr + src] (from each source) and
        # credits [(nn + ni)*nr + dst] (from each destination; start at 1: the
        # first put needs no credit)
        nn = len(names)
        self.names = {n: k for k, n in enumerate(names)}
        self.nn = nn
        self.flags = N.DeviceBuffer(16 * nr * max(nn, 1))
        self.expected = N.DeviceBuffer(16 * nr * max(nn, 1))
        self.counters = N.DeviceBuffer(4 * max(1, sum(len(rp.halo_rows(n)[0]) for n in names)))
        self.err = N.DeviceBuffer(8)              # first halo timeout: code, 0 = none
        for b in (self.expected, self.counters, self.err):
            N.check(L.ml_memset(b.ptr, 0, b.nbytes))
        init = np.concatenate([np.zeros(nr * max(nn, 1), np.uint64), np.ones(nr * max(nn, 1), np.uint64)])
        self.flags.upload(init)
        N.check(L.ml_synchronize())
        mine = {}
        for k in keys:
            h = (C.c_char * 64)()
            N.check(L.ml_ipc_handle(self.local[k].ptr, h), "ml_ipc_handle")
            mine[k] = bytes(h)
        fh = (C.c_char * 64)()
        N.check(L.ml_ipc_handle(self.flags.ptr, fh), "ml_ipc_handle")
        allh = transport.allgather_object({"bufs": mine, "flags": bytes(fh)})
        me = rp.rank
        ci = 0
        self.counter_of = {}
        for name in names:
            exports, _imp = rp.halo_rows(name)
            for dst in sorted(exports):
                h = allh[dst]["bufs"][(name, me)]
                self.remote[(name, dst)] = self._open(h)
                self.counter_of[(name, dst)] = self.counters.ptr + 4 * ci
                ci += 1
        peer_flags = {}
        for r in range(nr):
            if r != me and (any((n, r) in self.remote for n in names)
                            or any((n, r) in self.local for n in names)):
                peer_flags[r] = self._open(allh[r]["flags"])
        self.peer_flags = peer_flags

    def _delivery(self, ni: int, src: int) -> int:
        return 8 * (ni * self.rp.nranks + src)

    def _credit(self, ni: int, dst: int) -> int:
        return 8 * ((self.nn + ni) * self.rp.nranks + dst)

    def _open(self, handle: bytes) -> int:
        C, N = self.C, self.N
        p = C.c_void_p()
        N.check(N.lib().ml_ipc_open(C.create_string_buffer(handle, 64), C.byref(p)), "ml_ipc_open")
        self.opened.append(p.value)
        return p.value

    def put(self, name: str, index) -> int:
        """Enqueue the puts of one dat's export rows; returns the messages."""
        N, rp = self.N, self.rp
        from .device import dat_mirror
        d = rp.dats[name]
        m = dat_mirror(d)
        se, sc = m.strides(d)
        exports, _imports = rp.halo_rows(name)
        ni, me = self.names[name], rp.rank
        for dst, ids in sorted(exports.items()):
            N.check(N.lib().ml_wait_flag(self.flags.ptr + self._credit(ni, dst),
                                         self.expected.ptr + self._credit(ni, dst), self.timeout_ns,
                                         self.err.ptr, -(1 + ni * rp.nranks + dst)),
                    "ml_wait_flag")                    # dst has consumed our previous delivery
            N.check(N.lib().ml_put_rows(self.remote[(name, dst)], m.ptr, index(("e", name, dst), ids).ptr,
                                        ids.size, d.dim, se, sc, self.peer_flags[dst] + self._delivery(ni, me),
                                        self.counter_of[(name, dst)]), "ml_put_rows")
        return len(exports)

    def land(self, name: str, index, loop_index: int = 0) -> None:
        """Enqueue the waits and scatters of one dat's import rows."""
        N, rp = self.N, self.rp
        from .device import dat_mirror
        d = rp.dats[name]
        m = dat_mirror(d)
        se, sc = m.strides(d)
        _exports, imports = rp.halo_rows(name)
        ni, me = self.names[name], rp.rank
        for src, ids in sorted(imports.items()):
            code = 1 + (loop_index * self.nn + ni) * rp.nranks + src
            N.check(N.lib().ml_wait_flag(self.flags.ptr + self._delivery(ni, src),
                                         self.expected.ptr + self._delivery(ni, src), self.timeout_ns,
                                         self.err.ptr, code), "ml_wait_flag")
            N.check(N.lib().ml_unpack_rows(m.ptr, self.local[(name, src)].ptr, index(("i", name, src), ids).ptr,
                                           ids.size, d.dim, se, sc), "ml_unpack_rows")
            N.check(N.lib().ml_signal_flag(self.peer_flags[src] + self._credit(ni, me)), "ml_signal_flag")
        m.device_newer = True

    def check(self, loop_names) -> None:
        """Raise ExchangeTimeout (reference executor.py:343-359) if a wait expired."""
        code = np.zeros(1, np.int64)
        self.err.download(code)
        c = int(code[0])
        if not c:
            return
        from .executor import ExchangeTimeout
        nr, names = self.rp.nranks, sorted(self.names, key=self.names.get)
        if c < 0:
            k = -c - 1
            raise ExchangeTimeout(f"rank {self.rp.rank}: rank {k % nr} did not consume dat "
                                  f"{names[k // nr]!r} within {self.timeout_ns / 1e6:.0f} ms")
        k = c - 1
        src, ni, li = k % nr, (k // nr) % self.nn, k // (nr * self.nn)
        raise ExchangeTimeout(f"rank {self.rp.rank}: no message from rank {src} for dat {names[ni]!r} "
                              f"before loop {loop_names[li]!r} within {self.timeout_ns / 1e6:.0f} ms")

    def close(self):
        for p in self.opened:
            self.N.lib().ml_ipc_close(p)
        self.opened = []


class NvlinkReduce:
    """Reductions over NVLink peer memory: per reducing argument a gather
    buffer [nranks][dim] on every rank; ``ml_reduce_put`` stores this rank's
    partial into its row of every rank's buffer (IPC-mapped), and
    ``ml_reduce_fold`` waits for all rows and folds them in rank order onto
    the device-resident value — the result of the NCCL all-gather +
    ``ml_combine_ranks`` path, in two single-CTA kernels with no host or NCCL
    involvement (graph-capturable).  Credits keep a rank from overwriting a
    row the owner has not folded yet."""

    def __init__(self, rp: RankProgram, transport, timeout_ms: float = 10000.0):
        import ctypes as C
        from . import _native as N
        self.C, self.N, self.rp = C, N, rp
        L = N.lib()
        nr, me = rp.nranks, rp.rank
        self.timeout_ns = int(max(timeout_ms, 0.0) * 1e6)
        self.slot = {}                                    # id(part) -> (k, offset, nbytes)
        off = 0
        k = 0
        for reds in rp.reductions:
            for part, _val, _mode in reds:
                nb = part.buffer.nbytes
                self.slot[id(part)] = (k, off, nb)
                off += nr * nb
                k += 1
        self.nslot = k
        self.rows = N.DeviceBuffer(max(off, 8))
        self.cnt = N.DeviceBuffer(16 * nr * max(k, 1))    # deliveries [k][src], credits [k][dst]
        self.exp = N.DeviceBuffer(16 * nr * max(k, 1))
        self.err = N.DeviceBuffer(8)
        N.check(L.ml_memset(self.exp.ptr, 0, self.exp.nbytes))
        N.check(L.ml_memset(self.err.ptr, 0, 8))
        self.cnt.upload(np.concatenate([np.zeros(nr * max(k, 1), np.uint64),
                                        np.ones(nr * max(k, 1), np.uint64)]))
        N.check(L.ml_synchronize())
        hr, hc = (C.c_char * 64)(), (C.c_char * 64)()
        N.check(L.ml_ipc_handle(self.rows.ptr, hr), "ml_ipc_handle")
        N.check(L.ml_ipc_handle(self.cnt.ptr, hc), "ml_ipc_handle")
        allh = transport.allgather_object((bytes(hr), bytes(hc)))
        self.opened = []
        peer_rows, peer_cnt = {}, {}
        for r in range(nr):
            if r == me:
                peer_rows[r], peer_cnt[r] = self.rows.ptr, self.cnt.ptr
            else:
                peer_rows[r], peer_cnt[r] = self._open(allh[r][0]), self._open(allh[r][1])
        deliv = lambda kk, src: 8 * (kk * nr + src)                          # noqa: E731
        credit = lambda kk, dst: 8 * ((self.nslot + kk) * nr + dst)           # noqa: E731
        self.args = {}
        for pid, (kk, o, nb) in self.slot.items():
            rrow = np.array([peer_rows[r] + o + me * nb for r in range(nr)], np.uint64)
            rdel = np.array([peer_cnt[r] + deliv(kk, me) for r in range(nr)], np.uint64)
            rcre = np.array([peer_cnt[r] + credit(kk, me) for r in range(nr)], np.uint64)
            self.args[pid] = dict(rrow=_dev_array(rrow), rdel=_dev_array(rdel), rcre=_dev_array(rcre),
                                  credit=self.cnt.ptr + credit(kk, 0), credit_exp=self.exp.ptr + credit(kk, 0),
                                  deliv=self.cnt.ptr + deliv(kk, 0), deliv_exp=self.exp.ptr + deliv(kk, 0),
                                  rows=self.rows.ptr + o, k=kk)

    def _open(self, handle: bytes) -> int:
        C, N = self.C, self.N
        p = C.c_void_p()
        N.check(N.lib().ml_ipc_open(C.create_string_buffer(handle, 64), C.byref(p)), "ml_ipc_open")
        self.opened.append(p.value)
        return p.value

    def reduce(self, part, mode, partial_ptr: int, value_ptr: int, loop_index: int) -> None:
        N, rp = self.N, self.rp
        a = self.args[id(part)]
        code = 1 + loop_index * max(self.nslot, 1) + a["k"]
        N.check(N.lib().ml_reduce_put(partial_ptr, part.buffer.nbytes, a["rrow"].ptr, a["rdel"].ptr, a["credit"],
                                      a["credit_exp"], rp.nranks, self.timeout_ns, self.err.ptr, code),
                "ml_reduce_put")
        dt = 0 if np.dtype(part.dtype) == np.float64 else 1
        N.check(N.lib().ml_reduce_fold(value_ptr, a["rows"], a["deliv"], a["deliv_exp"], a["rcre"].ptr,
                                       rp.nranks, part.dim, {"INC": 3, "MIN": 4, "MAX": 5}[mode.name], dt,
                                       self.timeout_ns, self.err.ptr, code), "ml_reduce_fold")

    def check(self) -> None:
        code = np.zeros(1, np.int64)
        self.err.download(code)
        if int(code[0]):
            from .executor import ExchangeTimeout
            raise ExchangeTimeout(f"rank {self.rp.rank}: a reduction exchange did not complete within "
                                  f"{self.timeout_ns / 1e6:.0f} ms (code {int(code[0])})")

    def close(self):
        for p in self.opened:
            self.N.lib().ml_ipc_close(p)
        self.opened = []


def _dev_array(a: np.ndarray):
    from . import _native as N
    buf = N.DeviceBuffer(max(a.nbytes, 8))
    if a.nbytes:
        buf.upload(np.ascontiguousarray(a))
    return buf


class StreamRank:
    """Stream-ordered rank executor (the production multi-GPU path).

    Everything a program run does on a rank is enqueued on the library's
    compute stream without host round trips: loop launches (``ml_loop_run``),
    halo pack/unpack kernels, the transport's device collectives and the
    rank-ordered reduction fold (``ml_combine_ranks``).  Globals live in one
    device arena: one slot per running value (READ by later loops) and one
    per reducing argument (its rank-local partial); the arena image (user
    values + reduction identities) is uploaded once per run and the values
    are read back once at the end.

    Overlap (north star: "overlapping the exchange with core-element
    execution"): a gather-schedule loop that needs a halo exchange is split
    by target into *core* targets — no incident element reads an imported
    row — and *boundary* targets.  The export rows are packed, the transfer
    runs on a communication stream while the core launch runs on the compute
    stream, and the boundary launch waits on the transfer (CUDA events).  The
    two launches cover every target once, so the result is unchanged (the
    gather schedule accumulates each target in serial order either way)."""

    def __init__(self, rp: RankProgram, config, transport):
        import ctypes as C
        import torch
        from . import _native as N
        from .device import dat_mirror
        from .executor import _LoopEntry
        N.init(config.device_index())
        self.C, self.N, self.torch = C, N, torch
        self.rp, self.config, self.transport = rp, config, transport
        self.device = torch.device("cuda", config.device_index())
        self.lib_stream = torch.cuda.ExternalStream(N.lib().ml_stream(), device=self.device)
        self.comm_stream = torch.cuda.Stream(device=self.device)
        # globals arena: values, partials, rank-gather buffers (8-byte aligned slots)
        slots, off = {}, 0

        def slot(key, nbytes):
            nonlocal off
            slots[key] = off
            off += (nbytes + 255) // 256 * 256

        for gid, val in rp.values.items():
            slot(id(val), val.buffer.nbytes)
        for reds in rp.reductions:
            for part, _val, _mode in reds:
                slot(id(part), part.buffer.nbytes)
                slot(("gather", id(part)), part.buffer.nbytes * rp.nranks)
        self.arena = torch.zeros(max(off, 256), dtype=torch.uint8, device=self.device)
        self.image = torch.zeros(max(off, 256), dtype=torch.uint8).pin_memory()
        self.slots = slots
        base = self.arena.data_ptr()
        self.entries = [_LoopEntry(loop, rp.local, config, slots, base, rp.n_exec, rp.n_owned)
                        for loop in rp.loops]
        for e in self.entries:
            for d in e.dats:
                dat_mirror(d)
        self._splits: dict = {}
        self.split = [None] * len(self.entries)     # last split used by each loop (reporting)
        # exchange index lists and staging buffers up front (never inside a capture)
        for name in sorted({n for reads, _w in rp.roles for n in reads if n in rp.dats}):
            d = rp.dats[name]
            exports, imports = rp.halo_rows(name)
            for dst, ids in exports.items():
                self._index(("e", name, dst), ids)
                self._buf(("s", name, dst), ids.size * d.dim, d.dtype)
            for src, ids in imports.items():
                self._index(("i", name, src), ids)
                self._buf(("r", name, src), ids.size * d.dim, d.dtype)
        # halo path: direct NVLink stores (CUDA IPC) unless ML_HALO=nccl; every
        # rank must agree, so a failure anywhere falls back everywhere
        self.nvlink = None
        self.nvreduce = None
        self.halo_error = None
        if os.environ.get("ML_HALO", "p2p") == "p2p" and rp.nranks > 1:
            ok = 1
            try:
                self.nvlink = NvlinkHalo(rp, transport, config.timeout_ms)
                self.nvreduce = NvlinkReduce(rp, transport, config.timeout_ms)
            except Exception as ex:                     # noqa: BLE001 - reported, not hidden
                self.halo_error = f"{type(ex).__name__}: {ex}"[:200]
                ok = 0
            if min(transport.allgather_object(ok)) == 0:
                for x in (self.nvlink, self.nvreduce):
                    if x is not None:
                        x.close()
                self.nvlink = self.nvreduce = None
        global _LAST_HALO_PATH
        _LAST_HALO_PATH = "nvlink" if self.nvlink is not None else transport.name

    # -- setup ---------------------------------------------------------------------------
    def _split(self, i: int, names: tuple):
        """Core/boundary target descriptors of loop i (gather schedule) when the
        dats ``names`` are exchanged before it, or None (cached)."""
        key = (i, names)
        if key not in self._splits:
            self._splits[key] = self._build_split(i, names)
        return self._splits[key]

    def _build_split(self, i: int, names: tuple):
        e = self.entries[i]
        if (e.gather is None or (e.pfold is None and e.gather.nhub) or not names
                or e.loop.iter_set.size == 0):
            return None
        ex_names = set(names)
        loop = e.loop
        gathered = [a for a in loop.args if a.kind == "indirect" and a.mode is not READ]
        if any(a.dat.name in ex_names for a in gathered):
            return None
        if any(a.kind == "direct" and a.dat.name in ex_names for a in loop.args):
            return None
        bad_elem = np.zeros(e.n, dtype=bool)
        for a in loop.args:
            if a.kind == "indirect" and a.mode is READ and a.dat.name in ex_names:
                _ex, imports = self.rp.halo_rows(a.dat.name)
                if not imports:
                    continue
                imported = np.zeros(a.dat.set.size, dtype=bool)
                for ids in imports.values():
                    imported[ids] = True
                bad_elem |= imported[a.map.table[:e.n, a.slot]]
        if e.pfold is not None:
            return self._build_pfold_split(e, bad_elem)
        g = e.gather
        off = g.host["off"]
        deg = np.diff(off)
        bad_inc = bad_elem[g.host["elem"][:off[-1]]]
        per_target = np.add.reduceat(bad_inc.astype(np.int64), off[:-1]) if off[-1] else np.zeros(0)
        per_target = np.where(deg > 0, per_target, 0)
        idx = np.arange(g.ntargets)
        core, bnd = idx[per_target == 0], idx[per_target > 0]
        if core.size == 0 or bnd.size == 0:
            return None
        out = []
        for part in (core, bnd):
            sub = g.subset(part)
            desc = type(e.desc).from_buffer_copy(e.desc)
            desc.gather_ntargets = sub["ntargets"]
            desc.gather_off, desc.gather_elem = sub["off"].ptr, sub["elem"].ptr
            desc.gather_pos, desc.gather_targets = sub["pos"].ptr, sub["targets"].ptr
            desc.pf_rec = sub["rec"].ptr
            out.append((desc, sub))
        return out

    def _build_pfold_split(self, e, bad_elem: np.ndarray):
        """Primary fold: pass-1 rows none of whose elements read an imported row
        run first (overlapped with the exchange), without pass 2 or the hub
        folds; the other rows, the hub folds and pass 2 run after it."""
        pf = e.pfold
        h = pf.host
        off = h["off1"]
        if not off[-1]:
            return None
        bad = bad_elem[h["elem1"][:off[-1]]].astype(np.int64)
        per_row = np.add.reduceat(bad, off[:-1]) if off.size > 1 else np.zeros(0, np.int64)
        per_row = np.where(np.diff(off) > 0, per_row, 0)
        rows = np.arange(off.size - 1)
        core, bnd = rows[per_row == 0], rows[per_row > 0]
        if core.size == 0 or bnd.size == 0:
            return None
        out = []
        for k, part in enumerate((core, bnd)):
            sub = pf.pass1_subset(part)
            desc = type(e.desc).from_buffer_copy(e.desc)
            desc.pf_n1, desc.pf_off1 = sub["n1"], sub["off1"].ptr
            desc.pf_elem1, desc.pf_tl1 = sub["elem1"].ptr, sub["tl1"].ptr
            if sub["seg1"] is not None:
                desc.pf_seg1 = sub["seg1"].ptr
            if sub["rec"] is not None:
                desc.pf_rec = sub["rec"].ptr
            if k == 0:                 # pass 2 and the hub folds wait for every pass-1 row
                desc.pf_n2 = 0
                desc.pf_nhub1 = desc.pf_nhub2 = 0
            out.append((desc, sub))
        return out

    # -- one program run ------------------------------------------------------------------
    def _image(self, capturing: bool = False):
        ev = self.__dict__.get("_img_event")
        if ev is not None and not capturing:
            ev.synchronize()            # the previous run's copy has read the pinned image
        img = self.image.numpy()
        rp = self.rp
        for gid, val in rp.values.items():
            val.buffer[:] = rp.user_globals[gid].buffer
            o = self.slots[id(val)]
            img[o:o + val.buffer.nbytes] = val.buffer.view(np.uint8)
        for i, reds in enumerate(rp.reductions):
            for part, _val, mode in reds:
                ident = _identity(mode, part.dtype, part.dim)
                o = self.slots[id(part)]
                img[o:o + ident.nbytes] = ident.view(np.uint8)
        with self.torch.cuda.stream(self.lib_stream):
            self.arena.copy_(self.image, non_blocking=True)
        if not capturing:
            self._img_event = self.torch.cuda.Event()
            self._img_event.record(self.lib_stream)

    def _pack(self, name: str):
        N = self.N
        d = self.rp.dats[name]
        from .device import dat_mirror
        m = dat_mirror(d)
        se, sc = m.strides(d)
        exports, imports = self.rp.halo_rows(name)
        sends, recvs = {}, {}
        for dst, ids in exports.items():
            buf = self._buf(("s", name, dst), ids.size * d.dim, d.dtype)
            N.check(N.lib().ml_pack_rows(buf.data_ptr(), m.ptr, self._index(("e", name, dst), ids).ptr,
                                         ids.size, d.dim, se, sc), "ml_pack_rows")
            sends[dst] = buf
        for src, ids in imports.items():
            recvs[src] = self._buf(("r", name, src), ids.size * d.dim, d.dtype)
        return sends, recvs, (m, se, sc, imports, d)

    def _unpack(self, name: str, recvs, info):
        N = self.N
        m, se, sc, imports, d = info
        for src, ids in imports.items():
            N.check(N.lib().ml_unpack_rows(m.ptr, recvs[src].data_ptr(),
                                           self._index(("i", name, src), ids).ptr, ids.size, d.dim, se, sc),
                    "ml_unpack_rows")
        m.device_newer = True

    def _buf(self, key, n: int, dtype):
        cache = self.__dict__.setdefault("_bufs", {})
        torch = self.torch
        if key not in cache:
            tdt = torch.float64 if np.dtype(dtype) == np.float64 else torch.int64
            cache[key] = torch.empty(max(n, 1), dtype=tdt, device=self.device)
        return cache[key][:n]

    def _index(self, key, ids: np.ndarray):
        cache = self.__dict__.setdefault("_idx", {})
        if key not in cache:
            buf = self.N.DeviceBuffer(max(ids.nbytes, 4))
            if ids.size:
                buf.upload(np.ascontiguousarray(ids, dtype=np.int32))
            cache[key] = buf
        return cache[key]

    def _launch(self, desc) -> None:
        self.N.check(self.N.lib().ml_loop_run(self.C.byref(desc)), f"loop {desc.name!r}")

    def run(self, overlap: bool = True, capturing: bool = False) -> int:
        """Enqueue one program run; returns the halo messages sent.  With
        ``capturing`` (inside a CUDA-graph capture) no host synchronisation or
        timing event is issued."""
        torch, rp, tr = self.torch, self.rp, self.transport
        dirty = rp.__dict__.setdefault("dirty", {})
        messages = 0
        self._image(capturing)
        self.events = []
        for i, e in enumerate(self.entries):
            reads, writes = rp.roles[i]
            ev0 = None
            if not capturing:
                ev0 = torch.cuda.Event(enable_timing=True)
                ev0.record(self.lib_stream)
            names = [n for n in reads if dirty.get(n)]
            if self.nvlink is not None:
                for n in names:                         # peer stores start at once
                    messages += self.nvlink.put(n, self._index)
                split = self._split(i, tuple(names)) if overlap and names else None
                self.split[i] = split
                if split is not None:
                    self._launch(split[0][0])                   # core targets, overlapped
                for n in names:
                    self.nvlink.land(n, self._index, i)
                if split is not None:
                    self._launch(split[1][0])                   # boundary targets
                else:
                    self._launch(e.desc)
                packed = []
            else:
                packed = [(n, *self._pack(n)) for n in names]
                messages += sum(len(p[1]) for p in packed)
                split = self._split(i, tuple(names)) if overlap and packed else None
                self.split[i] = split
            if self.nvlink is not None:
                pass
            elif split is not None and tr.name == "nccl":
                ev_packed = torch.cuda.Event()
                ev_packed.record(self.lib_stream)
                self.comm_stream.wait_event(ev_packed)
                with torch.cuda.stream(self.comm_stream):
                    for n, sends, recvs, _info in packed:
                        tr.sendrecv_stream(sends, recvs)
                ev_moved = torch.cuda.Event()
                ev_moved.record(self.comm_stream)
                self._launch(split[0][0])                       # core targets, overlapped
                self.lib_stream.wait_event(ev_moved)
                for n, _sends, recvs, info in packed:
                    self._unpack(n, recvs, info)
                self._launch(split[1][0])                       # boundary targets
            else:
                for n, sends, recvs, info in packed:
                    tr.sendrecv_device(sends, recvs, self.lib_stream)
                    self._unpack(n, recvs, info)
                if split is not None:
                    self._launch(split[0][0])
                    self._launch(split[1][0])
                else:
                    self._launch(e.desc)
            for n in names:
                dirty[n] = False
            for part, val, mode in rp.reductions[i]:
                nbytes = part.buffer.nbytes
                po, go, vo = self.slots[id(part)], self.slots[("gather", id(part))], self.slots[id(val)]
                if self.nvreduce is not None:
                    base = self.arena.data_ptr()
                    self.nvreduce.reduce(part, mode, base + po, base + vo, i)
                    continue
                tr.allgather_device(self.arena[go:go + nbytes * rp.nranks], self.arena[po:po + nbytes],
                                    self.lib_stream)
                code = {"INC": 3, "MIN": 4, "MAX": 5}[mode.name]
                dt = 0 if np.dtype(part.dtype) == np.float64 else 1
                self.N.check(self.N.lib().ml_combine_ranks(self.arena.data_ptr() + vo,
                                                           self.arena.data_ptr() + go, rp.nranks,
                                                           part.dim, code, dt), "ml_combine_ranks")
            for n in writes:
                dirty[n] = True
            if not capturing:
                ev1 = torch.cuda.Event(enable_timing=True)
                ev1.record(self.lib_stream)
                self.events.append((ev0, ev1))
        for e in self.entries:
            for d in e.written:
                d._dev.device_newer = True
        if not capturing:
            self._ran = True
        return messages

    def capture(self, overlap: bool = True):
        """Capture one program run (loops, pack/unpack, NCCL exchanges and
        reductions, the overlap fork/join) as a CUDA graph on the compute
        stream; replay() then launches a whole rank step with one call (the
        host no longer paces the GPU).  NCCL transport only."""
        if self.transport.name != "nccl" and not (self.nvlink is not None and self.nvreduce is not None):
            raise ExecError("graph capture needs NCCL or the NVLink halo + reduction paths")
        torch = self.torch
        self.finish()
        if not self.__dict__.get("_ran"):
            raise ExecError("capture() needs one eager run first (steady halo pattern)")
        # build every core/boundary split the captured run will use (host + uploads),
        # replaying the dirty-bit evolution of one run without touching the device
        dirty = dict(self.rp.__dict__.get("dirty", {}))
        for i in range(len(self.entries)):
            reads, writes = self.rp.roles[i]
            names = [n for n in reads if dirty.get(n)]
            if names:
                self._split(i, tuple(names))
            for n in names:
                dirty[n] = False
            for n in writes:
                dirty[n] = True
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g, stream=self.lib_stream):
            msgs = self.run(overlap, capturing=True)
        self.graph, self.graph_messages = g, msgs
        return msgs

    def replay(self) -> int:
        with self.torch.cuda.stream(self.lib_stream):
            self.graph.replay()
        for e in self.entries:
            for d in e.written:
                d._dev.device_newer = True
        return self.graph_messages

    def loop_seconds(self) -> list:
        """Device time of each loop of the last run (exchange + launches + fold)."""
        return [a.elapsed_time(b) * 1e-3 for a, b in self.events]

    def finish(self) -> None:
        """Wait for the run and copy the running values back to the host."""
        global _LAST_OVERLAPPED
        _LAST_OVERLAPPED = [(e.loop.name, e.sched) for e, sp in zip(self.entries, self.split)
                            if sp is not None]
        self.N.check(self.N.lib().ml_synchronize(), "ml_synchronize")
        if self.nvlink is not None:
            self.nvlink.check([e.loop.name for e in self.entries])
        if self.nvreduce is not None:
            self.nvreduce.check()
        host = self.arena.cpu().numpy()
        for gid, val in self.rp.values.items():
            o = self.slots[id(val)]
            val.buffer[:] = host[o:o + val.buffer.nbytes].view(val.buffer.dtype)

    def sync_inputs(self) -> None:
        """Upload every local dat whose host payload is newer (after
        ``RankProgram.refresh_from_global``)."""
        from .device import dat_mirror
        for e in self.entries:
            for d in e.dats:
                dat_mirror(d)

    def close(self) -> None:
        """Unmap the peers' IPC buffers, then wait for every rank to have done
        so before this rank's exported buffers may be freed."""
        for x in (self.nvlink, self.nvreduce):
            if x is not None:
                x.close()
        self.nvlink = self.nvreduce = None
        self.transport.barrier()

    def launches_per_run(self) -> int:
        total = 0
        for i, e in enumerate(self.entries):
            if e.loop.iter_set.size == 0:
                continue
            base, colour = 0, False
            if e.pfold is not None:
                base = 1 + (1 if e.pfold.n2 > 0 else 0)
            elif e.gather is not None or not e.plan.has_writes:
                base = 1
            else:
                base, colour = e.plan.ncolors, True
            if self.split[i] is not None:
                base = 2
            if colour:      # k_combine per reduction (single-launch schedules fold in-kernel)
                total += sum(1 for a in e.loop.args if a.kind == "global" and a.mode.name != "READ")
            total += base
            total += 2 * len(self.rp.reductions[i])              # combine_ranks (+ gather is NCCL)
        return total


class _HostRows:
    """Numpy-side exchange for executors that expose pack/unpack (test oracle)."""

    @staticmethod
    def exchange_halo(dev, rp, name: str, transport) -> int:
        exports, imports = rp.halo_rows(name)
        d = rp.dats[name]
        sends = {dst: dev.pack(name, ids) for dst, ids in exports.items()}
        shapes = {src: (ids.size, d.dim) for src, ids in imports.items()}
        got = transport.exchange(sends, shapes, d.dtype)
        for src, ids in imports.items():
            dev.unpack(name, ids, got[src])
        return len(sends)


def _run_rank(rp: RankProgram, dev, transport, timeout_ms: float):
    """The rank main loop (reference executor.py:577-600) + reductions.  Dirty
    bits live on the RankProgram, so repeated runs keep halos coherent."""
    dirty = rp.__dict__.setdefault("dirty", {})
    messages = 0
    comm = np.zeros(len(rp.program))
    comp = np.zeros(len(rp.program))
    rp.refresh_globals()
    for i, loop in enumerate(rp.loops):
        reads, writes = rp.roles[i]
        t0 = time.perf_counter()
        for name in reads:
            if dirty.get(name):
                if hasattr(dev, "exchange_halo"):
                    messages += dev.exchange_halo(name, transport)
                else:
                    messages += _HostRows.exchange_halo(dev, rp, name, transport)
                dirty[name] = False
        t1 = time.perf_counter()
        dev.run_loop(i)
        for part, val, mode in rp.reductions[i]:
            parts = transport.allgather(part.buffer)
            val.buffer[:] = fold(val.buffer, parts, mode)
        comp[i] = time.perf_counter() - t1
        comm[i] = t1 - t0
        for name in writes:
            dirty[name] = True
    return messages, comm, comp


def init_distributed(config=None):
    """Initialise torch.distributed for one process per GPU (NCCL when GPUs are
    visible to torch, gloo otherwise); returns (rank, world, transport)."""
    import torch
    import torch.distributed as dist
    if not dist.is_initialized():
        use_nccl = torch.cuda.is_available() and os.environ.get("ML_TRANSPORT", "") != "gloo"
        if use_nccl:
            dev = int(os.environ.get("ML_DEVICE", os.environ.get("LOCAL_RANK", "0")))
            torch.cuda.set_device(dev)
            dist.init_process_group(backend="nccl", device_id=torch.device("cuda", dev))
        else:
            dist.init_process_group(backend="gloo")
    transport = NcclTransport() if dist.get_backend() == "nccl" else GlooTransport()
    return dist.get_rank(), dist.get_world_size(), transport


def setup_distributed(program, mesh, config, transport=None, executor_factory=None, layout=None):
    """Layout + this rank's local program + executor (one-time setup)."""
    import torch.distributed as dist
    rank, world, default_transport = init_distributed(config)
    if config.nranks not in (1, world):
        raise MeshError(f"nranks={config.nranks} but WORLD_SIZE={world}")
    if config.nranks != world:
        from dataclasses import replace
        config = replace(config, nranks=world)
    mesh.freeze()
    if config.chain_loops:             # fused pairs exchange the union of their halos
        from .chain import chain_program
        pinned = frozenset(config.block_size_table or ()) | frozenset(config.inc_schedule_table or ())
        program = chain_program(list(program), mesh, pinned)
    if layout is None:
        layout = build_layout(mesh, program, config)
    elif layout.nranks != world:
        raise MeshError(f"layout has {layout.nranks} ranks but WORLD_SIZE={world}")
    rp = RankProgram(mesh, program, layout, rank)
    transport = transport or default_transport
    if executor_factory:
        dev = executor_factory(rp, config)
    elif os.environ.get("ML_RANK_EXECUTOR", "stream") == "stream":
        dev = StreamRank(rp, config, transport)
    else:
        dev = DeviceRank(rp, config)
    return rp, dev, transport, layout, config


_DIST_CACHE_SIZE = 4


def _config_key(config) -> tuple:
    from dataclasses import fields
    out = []
    for f in fields(config):
        v = getattr(config, f.name)
        if isinstance(v, dict):
            v = tuple(sorted(v.items()))
        elif callable(v):
            v = id(v)
        out.append((f.name, v))
    return tuple(out)


def _cached_setup(program, mesh, config, transport, executor_factory, layout):
    """``setup_distributed`` once per (program, mesh version, config, layout):
    a repeated ``run_program`` (one call per time step) reuses the rank
    program, its device state and the opened IPC mappings, re-reading the
    local dats from the global mesh.  Evicted entries close their mappings
    (collectively: every rank makes the same calls in the same order)."""
    import torch.distributed as dist
    world = dist.get_world_size() if dist.is_initialized() else int(os.environ.get("WORLD_SIZE", "1"))
    cache = mesh.__dict__.setdefault("_ml_dist", OrderedDict())
    key = (tuple(id(l) for l in program), mesh.version, _config_key(config), world,
           id(layout) if layout is not None else None, id(executor_factory) if executor_factory else None,
           id(transport) if transport is not None else None)
    hit = cache.get(key)
    pinned = (layout, executor_factory, transport)
    if (hit is not None and len(hit[0]) == len(program)
            and all(a is b for a, b in zip(hit[0], program))
            and all(a is b for a, b in zip(hit[2], pinned))):
        cache.move_to_end(key)
        rp, dev = hit[1][0], hit[1][1]
        rp.refresh_from_global()
        if isinstance(dev, StreamRank):
            dev.sync_inputs()
        return hit[1]
    out = setup_distributed(program, mesh, config, transport, executor_factory, layout)
    cache[key] = (list(program), out, pinned)
    while len(cache) > _DIST_CACHE_SIZE:
        _, (_, old, _) = cache.popitem(last=False)
        if isinstance(old[1], StreamRank):
            old[1].close()
    return out


def run_program_distributed(program, mesh, config, transport=None, executor_factory=None,
                            layout=None, collector=None):
    """Owner-compute execution of a program on ``WORLD_SIZE`` processes (one GPU each)."""
    from .executor import RunResult
    from .perf import PerfCollector, useful_bytes
    t_start = time.perf_counter()
    rp, dev, transport, layout, config = _cached_setup(program, mesh, config, transport,
                                                       executor_factory, layout)
    if isinstance(dev, StreamRank):
        messages = dev.run()
        dev.finish()
        comp = np.array(dev.loop_seconds())
        comm = np.zeros_like(comp)
    else:
        messages, comm, comp = _run_rank(rp, dev, transport, config.timeout_ms)
    # final: every rank gets the owned rows of every dat, and the global values
    owned = {name: rp.owned_rows(name) for name in rp.dats}
    allowned = transport.allgather_object(owned)
    for name, gd in rp.global_dats.items():
        logical = gd.fetch()
        for r, ow in enumerate(allowned):
            ids = layout.sets[gd.set.name][r].owned
            logical[ids] = ow[name]
        gd.put(logical)
    for gid, val in rp.values.items():
        rp.user_globals[gid].buffer[:] = val.buffer
    msgs = sum(transport.allgather_object(messages))
    collector = collector if collector is not None else PerfCollector()
    for i, loop in enumerate(rp.program):
        collector.add(loop.name, float(comm[i] + comp[i]), useful_bytes(loop), comm=float(comm[i]),
                      comp=float(comp[i]))
    return RunResult(collector.finalize(), time.perf_counter() - t_start, messages=msgs,
                     layout=layout, assignments=layout.assignments)


def bench_distributed(args, metric, emit: bool = True, with_e2e: bool = True):
    """bench.py at N GPUs (torchrun, one process per GPU): same workload as N=1
    (strong scaling), RCB partition, halos over NCCL with the exchange
    overlapped with core targets (StreamRank).  ``value``: K program runs timed
    with CUDA events on each rank's compute stream, max over ranks.  ``e2e``:
    the same K runs through the host-resident path — every step uploads the
    rank's dats from pinned memory and downloads its owned rows of the written
    dats and the global values (wall clock, max over ranks).  Native banners
    (NCCL) are kept off stdout, which carries only the JSON line."""
    from .bench_support import stdout_to_stderr
    with stdout_to_stderr() as out:
        return _bench_distributed(args, metric, emit, with_e2e, out)


def _bench_distributed(args, metric, emit, with_e2e, out):
    import json
    import torch
    import torch.distributed as dist
    import paper_1403_7209_b200 as ml
    from . import _native as N  # noqa: F401
    from .bench_support import build_workload, clock_sampler, peaks_gbs
    from .device import pin_mesh
    rank, world, transport = init_distributed()
    mesh, prog, h, wname, setup = build_workload(args)
    edges = mesh.sets["edges"].size
    local_dev = int(os.environ.get("ML_DEVICE", os.environ.get("LOCAL_RANK", "0")))
    cfg = ml.BackendConfig(device=local_dev, nranks=world, partitioner="rcb", coord_dat="coords",
                           inc_schedule=("auto" if getattr(args, "inc_schedule", "auto") == "tuned"
                                         else args.inc_schedule))
    t0 = time.perf_counter()
    rp, dev, transport, layout, cfg = setup_distributed(prog, mesh, cfg, transport)
    setup["layout_and_local_mesh_s"] = round(time.perf_counter() - t0, 3)
    if not isinstance(dev, StreamRank):
        raise ExecError("bench_distributed needs the stream-ordered rank executor")
    for _ in range(max(args.warmup, 2)):
        dev.run()
    dev.finish()
    dev.run()                         # per-loop device times of one eager step (reported)
    dev.finish()
    loop_s = dev.loop_seconds()
    graphed = ((transport.name == "nccl" or (dev.nvlink is not None and dev.nvreduce is not None))
               and os.environ.get("ML_RANK_GRAPH", "1") == "1")
    graph_error = None
    if graphed:                       # one graph launch per rank step (NCCL inside)
        try:
            dev.capture()
        except Exception as ex:       # capture unsupported by this NCCL/torch: run eagerly
            graphed, graph_error = False, f"{type(ex).__name__}: {ex}"[:200]
            dev.finish()
    flags = torch.tensor([int(graphed)], device="cuda" if dist.get_backend() == "nccl" else "cpu")
    dist.all_reduce(flags, op=dist.ReduceOp.MIN)          # every rank must take the same path
    if graphed and not int(flags.item()):
        graphed = False
    step = dev.replay if graphed else dev.run
    dist.barrier()
    start, stop = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with clock_sampler(local_dev) as clk:
        time.sleep(0.3)
        for _ in range(max(3, args.steps)):                  # keep the GPU busy while sampling starts
            step()
        dev.finish()
        dist.barrier()
        msgs = 0
        start.record(dev.lib_stream)
        for _ in range(args.steps):
            msgs += step()
        stop.record(dev.lib_stream)
        dev.finish()
    dev_s = start.elapsed_time(stop) * 1e-3
    # end to end: host buffers in and out every step
    h2d = d2h = 0
    e2e_s = float("nan")
    if with_e2e:
        for d in rp.dats.values():
            d._pull()
        pin_mesh(rp.local)
        h2d = sum(d.nbytes for d in rp.dats.values())
        written = {d.name: d for e in dev.entries for d in e.written}
        d2h = sum(d.nbytes for d in written.values())
        from .device import dat_mirror
        dist.barrier()
        t_e2e = time.perf_counter()
        for _ in range(args.steps):
            for d in rp.dats.values():
                dat_mirror(d, force_upload=True)
            dev.run()
            dev.finish()
            for d in written.values():
                d._pull()
        e2e_s = time.perf_counter() - t_e2e
    t = torch.tensor([dev_s, e2e_s], dtype=torch.float64,
                     device="cuda" if dist.get_backend() == "nccl" else "cpu")
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    tmax, e2e_max = float(t[0].item()), float(t[1].item())
    # algorithmic bytes of one step summed over ranks (owned + exec-halo
    # elements, the reference convention executor.py:458-480)
    balg = torch.tensor([float(sum(e.alg for e in dev.entries))], dtype=torch.float64,
                        device="cuda" if dist.get_backend() == "nccl" else "cpu")
    dist.all_reduce(balg, op=dist.ReduceOp.SUM)
    balg_step = float(balg.item())
    halo = [len(layout.sets["nodes"][r].nonexec_halo) + len(layout.sets["nodes"][r].exec_halo)
            for r in range(world)]
    split = [e.loop.name for e, sp in zip(dev.entries, dev.split) if sp is not None]
    line = None
    if rank == 0:
        peak, src = peaks_gbs()
        line = {"metric": metric, "value": edges * args.steps / tmax, "unit": "edges/s",
                "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
                "ms_per_step": 1e3 * tmax / args.steps, "higher_is_better": True,
                "scaling": "strong", "vs_baseline": None, "dtype": "f64",
                "data": "synthetic (jittered 3-D grid, random numbering then CM renumbering)",
                "config": {"workload": wname, "edges": edges, "nodes": mesh.sets["nodes"].size,
                           "parallelism": f"owner-compute dp{world} (RCB)",
                           "transport": transport.name, "halo_nodes_per_rank": halo,
                           "halo_path": "nvlink-p2p (CUDA IPC peer stores)" if dev.nvlink is not None
                           else f"{transport.name} send/recv", "halo_p2p_error": dev.halo_error,
                           "reduction_path": "nvlink-p2p all-gather + rank-ordered fold"
                           if dev.nvreduce is not None else f"{transport.name} all-gather",
                           "overlapped_loops": split,
                           "cuda_graph": graphed, "cuda_graph_error": graph_error,
                           "l2": "per-rank working set streamed each step",
                           "timing": "CUDA events on each rank's compute stream around K runs, "
                                     "max over ranks", "setup": setup},
                "gpu_launches": dev.launches_per_run() * args.steps, "clocks": clk.summary(),
                "halo_messages_per_step": msgs / args.steps,
                "loops_ms_rank0": {e.loop.name: round(1e3 * t_, 4)
                                   for e, t_ in zip(dev.entries, loop_s)},
                "roofline": {"bound": "hbm", "kernel": "whole iteration (all ranks)",
                             "achieved": round(balg_step / (tmax / args.steps) / 1e9, 1),
                             "peak": round(world * peak, 1), "unit": "GB/s",
                             "frac": round(balg_step / (tmax / args.steps) / 1e9 / (world * peak), 4),
                             "traffic": None, "peak_source": src + f" x {world} GPUs",
                             "algorithmic_bytes_per_step": balg_step},
                "e2e": {"value": edges * args.steps / e2e_max, "unit": "edges/s",
                        "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": d2h,
                        "ms_per_step": 1e3 * e2e_max / args.steps,
                        "note": "rank 0's bytes; wall clock, max over ranks"},
                "cpu_baseline": None}
        if not with_e2e:
            line["e2e"] = None
        if emit:
            out.write_line(json.dumps(line))
    dist.barrier()
    dev.close()
    dist.destroy_process_group()
    return line
