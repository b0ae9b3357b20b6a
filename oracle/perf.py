"""Byte accounting oracle (TEST ORACLE ONLY).

``useful_bytes`` restates reference ``perf.py:30-47``: direct args move
``n*dim*itemsize*f``; each (dat, mode) group of indirect args moves
``#distinct targets * dim * itemsize * f``; globals ``dim*itemsize``;
f = 2 for RW/INC, else 1.  Map/index bytes are NOT counted.

``b_alg`` is the roofline byte model of SURVEY.md §8(d): ``useful_bytes``
plus 4 bytes (int32 device index) per iteration element per distinct
(map, column) pair used by indirect arguments.
"""
from __future__ import annotations

import numpy as np

__all__ = ["useful_bytes", "index_bytes", "b_alg"]


def _f(mode_name: str) -> int:
    return 2 if mode_name in ("RW", "INC") else 1


def useful_bytes(loop) -> int:
    n = loop.iter_set.size
    total = 0
    groups: dict = {}
    for a in loop.args:
        if a.kind == "global":
            total += a.glob.dim * a.glob.dtype.itemsize
        elif a.kind == "direct":
            total += n * a.dat.dim * a.dat.dtype.itemsize * _f(a.mode.name)
        else:
            groups.setdefault((a.dat.name, a.mode.name), []).append(a)
    for (_, mode), args in groups.items():
        if n == 0:
            continue
        distinct = np.unique(np.concatenate([a.map.table[:, a.slot] for a in args])).size
        d = args[0].dat
        total += distinct * d.dim * d.dtype.itemsize * _f(mode)
    return int(total)


def index_bytes(loop) -> int:
    cols = {(a.map.name, a.slot) for a in loop.args if a.kind == "indirect"}
    return 4 * loop.iter_set.size * len(cols)


def b_alg(loop) -> int:
    return useful_bytes(loop) + index_bytes(loop)
