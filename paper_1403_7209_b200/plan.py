"""Per-loop execution plans: blocking + two-level colouring, built natively.

Same contract as reference ``plan.py`` (``PlanConfig`` 25-27, ``ExecPlan``
30-45, ``build_plan`` 55-131, ``plan_for`` 138-148, ``plan_stats`` 151-153):
the plan is the race-freedom certificate the CUDA kernels consume — one
launch per block colour, element colours as ``__syncthreads``-separated
phases inside a CTA.  The colouring itself runs in C++
(``csrc/host_plan.cpp``, ``ml_plan_build``) and is bit-identical to the
reference's greedy first fit, including its per-dat offset quirk.

The device copy of a plan (block list ordered by colour, uint16 element
colours, per-block colour counts) is created on first GPU use and cached on
the plan object.
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass, field
from functools import cached_property

import numpy as np

from . import _native as N
from .core import Loop, Mesh, WRITE_MODES

__all__ = ["PlanConfig", "ExecPlan", "PlanStats", "build_plan", "plan_for", "plan_stats",
           "write_columns"]


@dataclass
class PlanConfig:
    block_size: int = 256


@dataclass
class ExecPlan:
    """Race-freedom certificate of one loop at one block size."""
    n: int
    block_size: int
    nblocks: int
    block_bounds: np.ndarray
    block_color: np.ndarray
    ncolors: int
    color_offsets: np.ndarray            # [ncolors+1] into blocks_flat
    blocks_flat: np.ndarray              # block ids ordered by colour
    elem_color: np.ndarray
    elem_ncolors: np.ndarray             # per block
    elem_order_flat: np.ndarray          # per block: elements by (colour, index)
    has_writes: bool = True
    max_elem_colors: int = 1
    _dev: object = field(default=None, repr=False, compare=False)

    @cached_property
    def blocks_by_color(self) -> list[np.ndarray]:
        o = self.color_offsets
        return [self.blocks_flat[o[c]:o[c + 1]] for c in range(self.ncolors)]

    @cached_property
    def block_elem_order(self) -> list[np.ndarray]:
        b = self.block_bounds
        return [self.elem_order_flat[b[i]:b[i + 1]] for i in range(self.nblocks)]

    def block_elements(self, b: int) -> np.ndarray:
        return np.arange(self.block_bounds[b], self.block_bounds[b + 1])


@dataclass
class PlanStats:
    nb: int
    nc: int
    blocks_per_color: list


def build_plan(n: int, write_cols: list, block_size: int) -> ExecPlan:
    """Plan ``n`` iterations whose indirect writes target ``write_cols``.

    ``write_cols``: one ``(dat key, 0-based target column)`` per indirect
    WRITE/RW/INC argument; targets of distinct keys never conflict.
    """
    if block_size < 1:
        raise ValueError(f"block size must be >= 1, got {block_size}")
    n = int(n)
    keys: dict = {}
    cols = [np.ascontiguousarray(c, dtype=np.int64) for _, c in write_cols]
    key_ids = np.array([keys.setdefault(k, len(keys)) for k, _ in write_cols], dtype=np.int32)
    col_ptrs = (C.c_void_p * max(len(cols), 1))(*[N.ptr(c) for c in cols])
    handle = C.c_void_p()
    L = N.lib()
    N.check(L.ml_plan_build(n, len(cols), col_ptrs,
                            key_ids.ctypes.data_as(C.POINTER(C.c_int32)) if len(cols) else None,
                            int(block_size), C.byref(handle)), "ml_plan_build")
    try:
        nb, nc, mx = C.c_int64(), C.c_int64(), C.c_int64()
        N.check(L.ml_plan_sizes(handle, C.byref(nb), C.byref(nc), C.byref(mx)))
        nb, nc = nb.value, nc.value
        block_color = np.empty(nb, np.int64)
        elem_nc = np.empty(nb, np.int64)
        offsets = np.empty(nc + 1, np.int64)
        flat = np.empty(nb, np.int64)
        elem_color = np.empty(n, np.int64)
        order = np.empty(n, np.int64)
        N.check(L.ml_plan_export(handle, N.ptr(block_color), N.ptr(elem_nc), N.ptr(offsets),
                                 N.ptr(flat), N.ptr(elem_color), N.ptr(order)), "ml_plan_export")
    finally:
        L.ml_plan_free(handle)
    bounds = np.minimum(np.arange(nb + 1, dtype=np.int64) * block_size, n)
    return ExecPlan(n, int(block_size), nb, bounds, block_color, nc, offsets, flat, elem_color,
                    elem_nc, order, has_writes=bool(cols) and n > 0, max_elem_colors=int(mx.value))


def write_columns(loop: Loop) -> list:
    """``(dat name, target column)`` per indirect write argument (plan.py:134-135)."""
    return [(a.dat.name, a.map.table[:, a.slot]) for a in loop.args
            if a.kind == "indirect" and a.mode in WRITE_MODES]


def plan_for(loop: Loop, mesh: Mesh, block_size: int | None = None, n: int | None = None) -> ExecPlan:
    """Build or fetch the cached plan (key: signature, block size, mesh version).

    ``n`` restricts the plan to the first ``n`` iteration elements (a rank's
    owned + exec-halo prefix on multi-GPU runs)."""
    bs = PlanConfig().block_size if block_size is None else int(block_size)
    key = (loop.signature(), bs, mesh.version) if n is None else (loop.signature(), bs, mesh.version, n)
    plan = mesh._plan_cache.get(key)
    if plan is None:
        cols = write_columns(loop)
        if n is not None:
            cols = [(k, c[:n]) for k, c in cols]
        plan = build_plan(loop.iter_set.size if n is None else n, cols, bs)
        mesh._plan_cache[key] = plan
        mesh._plan_builds += 1
    return plan


def plan_stats(plan: ExecPlan) -> PlanStats:
    return PlanStats(plan.nblocks, plan.ncolors, np.diff(plan.color_offsets).tolist())
