"""Per-element CPU executor: the reference semantics (TEST ORACLE ONLY).

Restates the reference serial backend (``executor.py:149-217``): the kernel
is applied to elements ``0..n-1`` in ascending order, receiving one
length-``dim`` numpy *view* per dat argument (an AOS row, or a strided SOA
column, so writes through the view land in the payload) and the global's
accumulator buffer itself for global arguments.  Also restates the
reduction helpers (``executor.py:115-143``) and the coloured-threads
schedule (``executor.py:223-275``) used as the CPU baseline.

Objects are duck-typed: anything with the reference attribute names works
(``loop.args``, ``arg.kind/mode/dat/map/slot/glob``, ``dat.data/dim/layout``,
``map.table``), so the same oracle runs on reference objects (to pin it)
and on the product's objects (to check the GPU).
"""
from __future__ import annotations

import numpy as np

__all__ = ["element_views", "run_loop", "run_program", "reduce_identity",
           "reduce_partials", "run_loop_coloured"]


def _mode(a) -> str:
    return a.mode.name


def _is_aos(dat) -> bool:
    return dat.layout.name == "AOS"


def element_views(loop, elements=None):
    """One accessor per argument: ``acc(e) -> view`` (executor.py:149-160, 193-203)."""
    out = []
    for a in loop.args:
        if a.kind == "global":
            buf = a.glob.buffer
            out.append(lambda e, buf=buf: buf)
            continue
        d = a.dat
        flat = d.data
        n = d.set.size
        target = a.map.table[:, a.slot] if a.kind == "indirect" else None
        if _is_aos(d):
            rows = flat.reshape(n, d.dim)
            out.append((lambda e, r=rows, t=target: r[t[e]]) if target is not None
                       else (lambda e, r=rows: r[e]))
        else:
            cols = flat.reshape(d.dim, n)
            out.append((lambda e, c=cols, t=target: c[:, t[e]]) if target is not None
                       else (lambda e, c=cols: c[:, e]))
    return out


def _apply(kernel, accessors, order, name):
    e = None
    try:
        for e in order:
            kernel(*[acc(e) for acc in accessors])
    except Exception as err:                                      # executor.py:181-183
        raise RuntimeError(f"kernel failed in loop {name!r} at element "
                           f"{'?' if e is None else int(e) + 1}: {err}") from err


def run_loop(loop) -> None:
    """Ascending-element application of one loop (executor.py:206-217)."""
    _apply(loop.kernel, element_views(loop), range(loop.iter_set.size), loop.name)


def run_program(program) -> None:
    for loop in program:
        run_loop(loop)


def reduce_identity(mode: str, dtype, dim: int) -> np.ndarray:
    """INC -> 0; MIN -> +inf / iinfo.max; MAX -> -inf / iinfo.min (executor.py:115-120)."""
    dtype = np.dtype(dtype)
    if mode == "INC":
        return np.zeros(dim, dtype=dtype)
    if dtype.kind == "i":
        fill = np.iinfo(dtype).max if mode == "MIN" else np.iinfo(dtype).min
    else:
        fill = np.inf if mode == "MIN" else -np.inf
    return np.full(dim, fill, dtype=dtype)


def reduce_partials(partials, mode: str, initial=None):
    """Strict left fold in the given order (executor.py:123-143)."""
    parts = [np.atleast_1d(np.asarray(p)) for p in partials]
    if initial is not None:
        acc = np.atleast_1d(np.asarray(initial)).copy()
    elif mode == "INC":
        acc = np.zeros_like(parts[0])
    else:
        acc, parts = parts[0].copy(), parts[1:]
    combine = {"INC": np.add, "MIN": np.minimum, "MAX": np.maximum}[mode]
    for p in parts:
        acc = combine(acc, p)
    return acc[0] if acc.size == 1 else acc


def run_loop_coloured(loop, plan) -> None:
    """The coloured schedule of executor.py:223-275, on one thread.

    Colours ascending, blocks of a colour in index order, elements of a block
    in ``block_elem_order``; each block reduces into its own identity
    scratch and the scratches fold onto the initial value in block order.
    (The reference runs blocks of one colour on a GIL-bound pool; the
    arithmetic order is the same.)
    """
    base = element_views(loop)
    red = [i for i, a in enumerate(loop.args)
           if a.kind == "global" and _mode(a) in ("INC", "MIN", "MAX")]
    parts = {i: [None] * plan.nblocks for i in red}
    for colour in range(plan.ncolors):
        for b in plan.blocks_by_color[colour]:
            b = int(b)
            acc = list(base)
            for i in red:
                g = loop.args[i].glob
                scratch = reduce_identity(_mode(loop.args[i]), g.dtype, g.dim)
                parts[i][b] = scratch
                acc[i] = lambda e, s=scratch: s
            _apply(loop.kernel, acc, plan.block_elem_order[b], loop.name)
    for i in red:
        a = loop.args[i]
        got = [p for p in parts[i] if p is not None]
        a.glob.buffer[:] = np.atleast_1d(reduce_partials(got, _mode(a),
                                                         initial=a.glob.buffer.copy()))
