"""Loop chaining: two consecutive loops over the same set run as one loop.

Hydra's ``iflux`` and ``vflux`` (the proxy's two edge loops) both gather the
two end nodes' ``q``/``x`` rows and increment both nodes' ``res``; run back to
back, each edge's node rows cross the L2→SM path twice and ``res`` is folded
twice.  A *chain* — declared natively next to the functors with
``ML_REGISTER_CHAIN(first, second, fused, Functor)`` — says the pair may run
as one loop of a fused functor that evaluates the first kernel then the
second on each element.  This module decides, per program, where that is
legal and builds the fused :class:`~paper_1403_7209_b200.core.Loop`.

Legality (a chained pair must give the result of running the loops in
order, up to the order of floating-point increments):

* the loops are adjacent in the program and iterate over the same set;
* a global one loop reduces (INC/MIN/MAX) does not appear in the other (a
  reduction read by the second loop would see a partial value); READ
  globals may appear in both;
* at most one of the two kernels takes constants (the fused functor hands
  the same constant block to both halves);
* every dat both loops touch is READ in both, or INC in both (increments
  commute); a dat one loop writes any other way does not appear in the other
  loop at all;
* the fused functor takes every argument of the first loop, and every
  argument of the second loop it does not list is identical (dat, map, slot,
  mode) to one of the first loop's.

For integer data the chained result is bit-identical to the sequential one;
for floating point the per-target increment order interleaves the two
loops' contributions (each target still receives them in element order), so
parity is the reference's rtol 1e-12 criterion, not bitwise.  The reference
has no loop chaining (its executors run ``program`` loop by loop,
``executor.py:707-729``); this is a B200 schedule, off with
``BackendConfig(chain_loops=False)``.
"""
from __future__ import annotations

import ctypes as C
from collections import OrderedDict

from . import _native as N
from .core import INC, READ, Loop, Mesh
from .kernels import KernelBinding, resolve_kernel

__all__ = ["chain_lookup", "chain_program", "chain_pair"]

_CHAIN_CACHE_SIZE = 256          # adjacent pairs remembered per mesh


def chain_lookup(first: str, second: str):
    """(fused functor, fused position of each first-loop argument, of each
    second-loop argument) or None."""
    buf = C.create_string_buffer(128)
    na, nb = C.c_int32(), C.c_int32()
    apos, bpos = (C.c_int32 * 64)(), (C.c_int32 * 64)()
    rc = N.lib().ml_chain_lookup(first.encode(), second.encode(), buf, len(buf), C.byref(na), apos,
                                 C.byref(nb), bpos)
    if rc != 0:
        return None
    return buf.value.decode(), list(apos[:na.value]), list(bpos[:nb.value])


def _same(a, b) -> bool:
    return (a.kind == b.kind and a.mode is b.mode and a.dat is b.dat and a.map is b.map
            and a.slot == b.slot)


def _hazard_free(A: Loop, B: Loop) -> bool:
    for X, Y in ((A, B), (B, A)):
        for a in X.args:              # a reduced global stays private to its loop
            if a.kind == "global" and a.mode is not READ and any(b.glob is a.glob for b in Y.args):
                return False
    for a in A.args:
        for b in B.args:
            if a.kind == "global" or b.kind == "global" or a.dat is not b.dat:
                continue
            if not ((a.mode is READ and b.mode is READ) or (a.mode is INC and b.mode is INC)):
                return False
    return True


def chain_pair(A: Loop, B: Loop) -> Loop | None:
    """The fused loop for A followed by B, or None when no legal chain exists."""
    if A.iter_set is not B.iter_set or not _hazard_free(A, B):
        return None
    try:
        ba, bb = resolve_kernel(A.kernel), resolve_kernel(B.kernel)
    except Exception:
        return None
    if (ba.fconsts or ba.iconsts) and (bb.fconsts or bb.iconsts):
        return None                   # the fused functor passes one constant block to both
    hit = chain_lookup(ba.functor, bb.functor)
    if hit is None:
        return None
    fused, apos, bpos = hit
    if len(apos) != len(A.args) or len(bpos) != len(B.args):
        return None
    nf = max(apos + bpos, default=-1) + 1
    slots: list = [None] * nf
    for arg, k in list(zip(A.args, apos)) + list(zip(B.args, bpos)):
        if not 0 <= k < nf:
            return None
        if slots[k] is None:
            slots[k] = arg
        elif not _same(slots[k], arg):         # the functor reads one row for both
            return None
    if any(s is None for s in slots):
        return None
    from .executor import _loop_dtype
    fid = C.c_int32()
    for L in (A, B):                  # the fused functor must exist for the loops' type
        if N.lib().ml_functor_lookup(fused.encode(), _loop_dtype(L), C.byref(fid)) != 0:
            return None
    fa, fb = A.kernel, B.kernel

    def kernel(*views):
        fa(*[views[k] for k in apos])
        fb(*[views[k] for k in bpos])

    kernel.__ml_binding__ = KernelBinding(fused, ba.fconsts or bb.fconsts, ba.iconsts or bb.iconsts)
    kernel.__qualname__ = f"chain[{ba.functor}+{bb.functor}]"
    return Loop(f"{A.name}+{B.name}", A.iter_set, slots, kernel)


def chain_program(program: list[Loop], mesh: Mesh, pinned=frozenset()) -> list[Loop]:
    """``program`` with every legal adjacent chained pair replaced by its
    fused loop (left to right; fused loops are cached on the mesh so a
    program's compiled form stays valid across calls).  Loops named in
    ``pinned`` — those a per-loop table (block size, INC schedule) names —
    are never fused, so the table entry applies to the loop as written."""
    cache = mesh.__dict__.setdefault("_ml_chains", OrderedDict())
    out: list[Loop] = []
    i = 0
    while i < len(program):
        if i + 1 < len(program) and program[i].name not in pinned and program[i + 1].name not in pinned:
            A, B = program[i], program[i + 1]
            key = (id(A), id(B))
            hit = cache.get(key)
            if hit is None or hit[0] is not A or hit[1] is not B:
                hit = (A, B, chain_pair(A, B))
                cache[key] = hit
                while len(cache) > _CHAIN_CACHE_SIZE:
                    cache.popitem(last=False)
            else:
                cache.move_to_end(key)
            if hit[2] is not None:
                out.append(hit[2])
                i += 2
                continue
        out.append(program[i])
        i += 1
    return out
