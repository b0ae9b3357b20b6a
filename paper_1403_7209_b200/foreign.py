"""Programs built with the reference package's own objects, run on B200.

North_star asks that Hydra-style solver code written against the reference
``meshloop`` package runs unchanged.  Such code builds ``meshloop.Mesh`` /
``Dat`` / ``Map`` / ``Global`` / ``Loop`` objects (reference
``core.py:97-317``) and calls ``meshloop.run_program`` (``executor.py:707-729``).
The reference classes declare ``__slots__`` (``Dat``: name, set, dim,
dtype, layout, data — ``core.py:131-139``), so the backend cannot hang its
device mirrors on them.  Instead every reference mesh gets a *shadow*: a
product :class:`~paper_1403_7209_b200.core.Mesh` whose maps and dats share
the reference objects' numpy arrays (no copy), kept in a side table keyed
weakly by the reference mesh.  A reference program is translated once per
program (cached) into product loops over the shadow, with one shadow
``Global`` per reference ``Global`` sharing its ``buffer`` (so a MIN one loop
reduces is READ by the next on the device, and results land in the
reference's own buffer).

Coherence follows the reference's contract that ``dat.data`` is the truth
between runs: each run re-binds any payload the caller replaced (e.g. by
``meshloop.transform_layout``, which assigns a new array, ``core.py:179-192``),
uploads every dat the program reads, and downloads every dat it writes back
into the reference arrays in place — the same host-residency path that
``bench.py``'s ``e2e`` measures.  A renumbering of the reference mesh bumps
its ``version`` (``renumber.py:141-166``) and rebuilds the shadow.

Two ways in:

* ``paper_1403_7209_b200.run_program(program, ref_mesh, config)`` — the
  branch ``INTEGRATION.md`` shows; ``config`` may be this package's
  ``BackendConfig`` or the reference's (its common fields are carried over);
* :func:`install` — registers ``"cuda"`` in the reference's backend switch
  (``executor.py:50``) so the stock call
  ``meshloop.run_program(program, mesh, meshloop.BackendConfig(backend="cuda"))``
  runs on B200; every other backend still runs the reference's own code.
"""
from __future__ import annotations

import weakref
from collections import OrderedDict
from dataclasses import fields, replace

import numpy as np

from . import core
from .core import ExecError

__all__ = ["is_foreign_mesh", "shadow_mesh", "run_foreign", "install", "to_backend_config",
           "export_mesh", "export_program"]

_SHADOWS: "weakref.WeakKeyDictionary" = weakref.WeakKeyDictionary()
_PROGRAMS_PER_MESH = 32

#: reference BackendConfig fields (executor.py:59-75) that carry over
_SHARED_FIELDS = ("nthreads", "nranks", "block_size", "block_size_table", "partitioner",
                  "coord_dat", "balance", "class_a_ranks", "class_a_width", "class_b_width",
                  "class_a_speed", "class_b_speed", "timeout_ms", "simulated_elem_cost",
                  "cost_model", "phase_callback")


def is_foreign_mesh(mesh) -> bool:
    """True for a mesh that is not this package's (e.g. a reference ``meshloop.Mesh``)."""
    return not isinstance(mesh, core.Mesh)


def _layout(lay) -> core.Layout:
    return core.SOA if getattr(lay, "name", str(lay)).upper() == "SOA" else core.AOS


class _Shadow:
    """Product mesh sharing one reference mesh's arrays, plus its translated programs."""

    def __init__(self, ref):
        self.ref = weakref.ref(ref)
        self.version = ref.version
        pm = core.Mesh(auto_soa_threshold=ref.auto_soa_threshold)
        for name, s in ref.sets.items():
            pm.sets[name] = core.Set(name, s.size)
        for name, m in ref.maps.items():
            table = m.table
            if table.dtype != np.int64 or table.shape != (m.from_set.size, m.arity):
                table = np.asarray(table, dtype=np.int64).reshape(m.from_set.size, m.arity)
            pm.maps[name] = core.Map(name, pm.sets[m.from_set.name], pm.sets[m.to_set.name],
                                     m.arity, table)
        for name, d in ref.dats.items():
            pm.dats[name] = core.Dat(name, pm.sets[d.set.name], d.dim, np.dtype(d.dtype),
                                     _layout(d.layout), d.data)
        pm.version = ref.version
        self.mesh = pm
        self.programs: OrderedDict = OrderedDict()

    # -- identity checks: a reference object must be the one this mesh declared --
    def _set(self, ref, s):
        if ref.sets.get(s.name) is not s:
            raise ExecError(f"set {s.name!r} is not declared on this mesh")
        return self.mesh.sets[s.name]

    def _dat(self, ref, d):
        if ref.dats.get(d.name) is not d:
            raise ExecError(f"dat {d.name!r} is not declared on this mesh")
        return self.mesh.dats[d.name]

    def _map(self, ref, m):
        if ref.maps.get(m.name) is not m:
            raise ExecError(f"map {m.name!r} is not declared on this mesh")
        return self.mesh.maps[m.name]

    def translate(self, ref, program) -> tuple[list, list]:
        """Product loops of a reference program and its (reference, shadow) globals."""
        key = tuple(id(l) for l in program)
        hit = self.programs.get(key)
        if hit is not None and len(hit[0]) == len(program) and all(
                a is b for a, b in zip(hit[0], program)):
            self.programs.move_to_end(key)
            return hit[1], hit[2]
        globs: dict = {}
        loops = []
        for l in program:
            args = []
            for a in l.args:
                mode = core.AccessMode[a.mode.name]
                if a.kind == "global":
                    pair = globs.get(id(a.glob))
                    if pair is None:
                        g = core.Global.__new__(core.Global)
                        g.name, g.buffer, g._dev = a.glob.name, a.glob.buffer, None
                        pair = globs[id(a.glob)] = (a.glob, g)
                    args.append(core.arg_global(pair[1], mode))
                elif a.kind == "direct":
                    args.append(core.arg_direct(self._dat(ref, a.dat), mode))
                elif a.kind == "indirect":
                    args.append(core.arg_indirect(self._dat(ref, a.dat), self._map(ref, a.map),
                                                  a.slot + 1, mode))
                else:
                    raise ExecError(f"loop {l.name!r}: unknown argument kind {a.kind!r}")
            loops.append(core.Loop(l.name, self._set(ref, l.iter_set), args, l.kernel))
        entry = (list(program), loops, list(globs.values()))
        self.programs[key] = entry
        while len(self.programs) > _PROGRAMS_PER_MESH:
            self.programs.popitem(last=False)
        return loops, entry[2]

    def sync_in(self, ref, globs) -> None:
        """The reference arrays are authoritative: re-bind replaced payloads and
        mark every payload host-newer (the caller may have written it in place)."""
        for name, rd in ref.dats.items():
            pd = self.mesh.dats[name]
            lay = _layout(rd.layout)
            if pd._host is not rd.data or pd.layout is not lay:
                pd.layout = lay
                pd.data = rd.data
            else:
                pd._host_modified()
        for rg, pg in globs:
            if pg.buffer is not rg.buffer:
                pg.buffer = rg.buffer

    def sync_out(self) -> None:
        """Pull every device-newer payload into the shared reference arrays."""
        for pd in self.mesh.dats.values():
            pd._pull()


def shadow_mesh(ref) -> _Shadow:
    """The (cached) shadow of reference mesh ``ref``; rebuilt after a renumbering."""
    sh = _SHADOWS.get(ref)
    if sh is None or sh.version != ref.version or set(sh.mesh.dats) != set(ref.dats):
        sh = _SHADOWS[ref] = _Shadow(ref)
    return sh


def to_backend_config(config):
    """This package's ``BackendConfig`` for ``config`` (ours, the reference's, or None)."""
    from .executor import BackendConfig
    if config is None:
        return BackendConfig()
    if isinstance(config, BackendConfig):
        return config
    ours = {f.name for f in fields(BackendConfig)}
    kw = {k: getattr(config, k) for k in _SHARED_FIELDS if k in ours and hasattr(config, k)}
    return BackendConfig(**kw)


def run_foreign(program, mesh, config=None):
    """Run a program of reference objects on B200 (see the module docstring)."""
    from .executor import run_program
    cfg = to_backend_config(config)
    sh = shadow_mesh(mesh)
    loops, globs = sh.translate(mesh, list(program))
    sh.sync_in(mesh, globs)
    mesh.freeze()                         # reference run_serial/run_program freeze (executor.py:209)
    sh.mesh._frozen = True
    result = run_program(loops, sh.mesh, replace(cfg, residency="host"))
    sh.sync_out()
    return result


def install(meshloop_module=None):
    """Add ``"cuda"`` to the reference's backend switch (``executor.py:50``,
    validated at ``78-79``): ``meshloop.run_program`` with
    ``BackendConfig(backend="cuda")`` then runs here; other backends are untouched.
    Returns the patched module.  Idempotent."""
    if meshloop_module is None:
        import meshloop as meshloop_module
    ex = meshloop_module.executor
    if "cuda" not in ex._BACKENDS:
        ex._BACKENDS = (*ex._BACKENDS, "cuda")
    if not getattr(ex.run_program, "__ml_b200__", False):
        stock = ex.run_program

        def run_program(program, mesh, config=None):
            if config is not None and getattr(config, "backend", None) == "cuda":
                return run_foreign(program, mesh, config)
            return stock(program, mesh, config)

        run_program.__ml_b200__ = True
        run_program.__wrapped__ = stock
        run_program.__doc__ = stock.__doc__
        ex.run_program = run_program
        meshloop_module.run_program = run_program
    return meshloop_module


_DEFAULT = object()


def export_mesh(mesh: core.Mesh, api, auto_soa_threshold=_DEFAULT):
    """Declare ``mesh``'s sets, maps and dats (same values) on a new mesh of
    package ``api`` (e.g. the reference ``meshloop``) through that package's own
    ``decl_*`` calls, so its validation and auto-SOA policy apply
    (``core.py:362-407``).  Used to hand meshes generated here to the stock
    reference (bench.py's reference arm, the reference-object parity tests)."""
    thr = mesh.auto_soa_threshold if auto_soa_threshold is _DEFAULT else auto_soa_threshold
    out = api.Mesh(auto_soa_threshold=thr)
    sets = {n: out.decl_set(n, s.size) for n, s in mesh.sets.items()}
    for n, m in mesh.maps.items():
        out.decl_map(n, sets[m.from_set.name], sets[m.to_set.name], m.arity,
                     (m.table + 1).reshape(-1))
    for n, d in mesh.dats.items():
        out.decl_dat(n, sets[d.set.name], d.dim, d.dtype.name, d.fetch().reshape(-1))
    return out


def export_program(program, ref, api):
    """``program`` (loops over a product mesh) as loops of package ``api`` over
    ``ref`` — a mesh exported from it by :func:`export_mesh` (matched by name);
    each product ``Global`` becomes one fresh ``api.Global`` with the same values."""
    gmap: dict = {}
    loops = []
    for l in program:
        args = []
        for a in l.args:
            mode = getattr(api, a.mode.name)
            if a.kind == "global":
                g = gmap.get(id(a.glob))
                if g is None:
                    g = gmap[id(a.glob)] = api.Global(a.glob.buffer.copy(), name=a.glob.name)
                args.append(api.arg_global(g, mode))
            elif a.kind == "direct":
                args.append(api.arg_direct(ref.dats[a.dat.name], mode))
            else:
                args.append(api.arg_indirect(ref.dats[a.dat.name], ref.maps[a.map.name], a.slot + 1, mode))
        loops.append(api.Loop(l.name, ref.sets[l.iter_set.name], args, l.kernel))
    return loops
