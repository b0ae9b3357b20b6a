"""OP2-style spellings of the API (paper §3, Figs. 3-4).

    from paper_1403_7209_b200.op2 import *
    op_init()
    nodes = op_decl_set(14, "nodes")
    cells = op_decl_set(17, "cells")
    pcell = op_decl_map(cells, nodes, 3, c_to_n, "pcell")          # 1-based, as Fortran
    areac = op_decl_dat(cells, 1, "r8", ca_data, "c_area")
    arean = op_decl_dat(nodes, 1, "r8", na_data, "n_area")
    op_par_loop(cells, distr,
                op_arg_dat(areac, -1, OP_ID, 1, "r8", OP_READ),
                op_arg_dat(arean, 1, pcell, 1, "r8", OP_INC),
                op_arg_dat(arean, 2, pcell, 1, "r8", OP_INC),
                op_arg_dat(arean, 3, pcell, 1, "r8", OP_INC))

Each call maps onto the meshloop API: ``op_decl_*`` ->
``Mesh.decl_*`` on the session mesh, ``op_arg_dat`` -> ``arg_direct`` (index
-1 / ``OP_ID``) or ``arg_indirect`` (1-based index), ``op_arg_gbl`` ->
``arg_global`` and ``op_par_loop`` builds the ``Loop`` and executes it at
once on the session's B200 backend; device state persists between calls,
so a sequence of ``op_par_loop`` calls is a solver.
"""
from __future__ import annotations

import numpy as np

from .core import (INC, MAX, MIN, READ, RW, WRITE, DeclError, Global, Loop, LoopError, Mesh,
                   arg_direct, arg_global, arg_indirect)
from .executor import BackendConfig, run_program

__all__ = ["OP_READ", "OP_WRITE", "OP_RW", "OP_INC", "OP_MIN", "OP_MAX", "OP_ID", "op_init",
           "op_exit", "op_decl_set", "op_decl_map", "op_decl_dat", "op_decl_const", "op_arg_dat",
           "op_arg_gbl", "op_par_loop", "op_fetch_data", "op_mesh"]

OP_READ, OP_WRITE, OP_RW, OP_INC, OP_MIN, OP_MAX = READ, WRITE, RW, INC, MIN, MAX


class _OpId:
    """The identity map of direct arguments."""

    def __repr__(self):
        return "OP_ID"


OP_ID = _OpId()

_TYPES = {"r8": "float64", "double": "float64", "real(8)": "float64", "float64": "float64",
          "i8": "int64", "int": "int64", "integer(8)": "int64", "int64": "int64"}

_session: dict = {}


def op_init(config: BackendConfig | None = None, mesh: Mesh | None = None) -> Mesh:
    """Start a session (one mesh, one backend configuration)."""
    _session["mesh"] = mesh if mesh is not None else Mesh()
    _session["config"] = config or BackendConfig()
    _session["gbl"] = []
    return _session["mesh"]


def op_exit() -> None:
    _session.clear()


def op_mesh() -> Mesh:
    if "mesh" not in _session:
        op_init()
    return _session["mesh"]


def _kind(type_: str) -> str:
    try:
        return _TYPES[type_]
    except KeyError:
        raise DeclError(f"unsupported OP2 type {type_!r}; use 'r8' or 'i8'") from None


def op_decl_set(size: int, name: str):
    return op_mesh().decl_set(name, size)


def op_decl_map(from_set, to_set, dim: int, data, name: str):
    """``data``: flat, 1-based (the Fortran convention of Fig. 3)."""
    return op_mesh().decl_map(name, from_set, to_set, dim, data)


def op_decl_dat(set_, dim: int, type_: str, data, name: str):
    return op_mesh().decl_dat(name, set_, dim, _kind(type_), data)


def op_decl_const(dim: int, type_: str, data, name: str) -> None:
    """Scalar constants only (the reference's constants table holds scalars)."""
    vals = np.atleast_1d(np.asarray(data, dtype=_kind(type_)))
    if dim != 1 or vals.size != 1:
        raise DeclError(f"constant {name!r}: only scalar constants (dim 1) are supported")
    op_mesh().set_constant(name, vals[0].item())


def op_arg_dat(dat, idx: int, map_, dim: int, type_: str, acc):
    """Direct when ``idx == -1`` / ``map is OP_ID``; else column ``idx`` (1-based)."""
    if dim != dat.dim or np.dtype(_kind(type_)) != dat.dtype:
        raise LoopError(f"op_arg_dat({dat.name}): declared dim/type {dim}/{type_} do not match "
                        f"the dat ({dat.dim}/{dat.dtype.name})")
    if map_ is OP_ID or idx == -1:
        return arg_direct(dat, acc)
    return arg_indirect(dat, map_, idx, acc)


def op_arg_gbl(data, dim: int, type_: str, acc):
    """A global: a :class:`Global`, or a numpy array updated in place after the loop."""
    if isinstance(data, Global):
        g = data
    else:
        arr = np.asarray(data)
        g = Global(arr.astype(_kind(type_), copy=True).reshape(-1)[:dim], name="gbl")
        if isinstance(data, np.ndarray):
            _session.setdefault("gbl", []).append((data, g))
    if g.dim != dim:
        raise LoopError(f"op_arg_gbl: dim {dim} but the global holds {g.dim} values")
    return arg_global(g, acc)


def op_par_loop(*call, name: str | None = None):
    """Build the loop and run it now on the session backend; returns its RunResult.

    Both OP2 spellings: ``op_par_loop(set, kernel, *args)`` (Fortran, Fig. 4)
    and ``op_par_loop(kernel, "name", set, *args)`` (C++).
    """
    if call and callable(call[0]):
        kernel, name, set_, args = call[0], call[1], call[2], call[3:]
    else:
        set_, kernel, args = call[0], call[1], call[2:]
    loop = Loop(name or getattr(kernel, "__name__", "op_par_loop"), set_, list(args), kernel)
    result = run_program([loop], op_mesh(), _session.get("config") or BackendConfig())
    for arr, g in _session.pop("gbl", []):
        arr.reshape(-1)[:g.dim] = g.buffer
    _session["gbl"] = []
    return result


def op_fetch_data(dat) -> np.ndarray:
    return dat.fetch()
