"""Partition and owner-compute halo oracle (TEST ORACLE ONLY).

Restates reference ``partition.py``:

* ``trivial`` (44-51): contiguous ranges, the first ``size % nranks`` ranks
  one element larger;
* ``rcb`` (81-106): power-of-two ranks, 2-D/3-D; recursive, axis = depth %
  dim; elements ordered by (coordinate, element id); the LOWER half takes
  ``ceil(len/2)``;
* ``derive`` (109-140): iteration sets with indirect arguments follow the
  owner of column 0 of their first loop's first indirect map; others trivial;
* ``halos`` (186-260): exec halo of iteration set on rank r = foreign
  elements with an indirect WRITE/RW/INC target owned by r; non-exec halo
  = foreign targets referenced by executed (owned + exec) elements that
  are not already in r's exec halo; imports = halo ids ascending grouped by
  owner; exports mirror imports exactly.

Inputs are plain arrays: ``loops`` is a list of dicts
``{"iter": set name, "args": [(kind, mode name, target set | None,
target column | None, full map table | None)]}``.
"""
from __future__ import annotations

import numpy as np

__all__ = ["trivial", "rcb", "derive", "halos"]


def trivial(size: int, nranks: int) -> np.ndarray:
    out = []
    q, rem = divmod(size, nranks)
    for r in range(nranks):
        out += [r] * (q + (1 if r < rem else 0))
    return np.array(out, dtype=np.int64)


def rcb(points: np.ndarray, nranks: int) -> np.ndarray:
    pts = np.asarray(points, dtype=np.float64)
    dim = pts.shape[1]
    owner = np.zeros(pts.shape[0], dtype=np.int64)

    def split(ids, first, parts, depth):
        if parts == 1:
            for e in ids:
                owner[e] = first
            return
        ax = depth % dim
        ranked = sorted(ids, key=lambda e: (pts[e, ax], e))
        cut = (len(ranked) + 1) // 2
        split(ranked[:cut], first, parts // 2, depth + 1)
        split(ranked[cut:], first + parts // 2, parts // 2, depth + 1)

    split(list(range(pts.shape[0])), 0, nranks, 0)
    return owner


def derive(loops, base: dict, sizes: dict, nranks: int) -> dict:
    """Complete ``base`` (set -> owner array) over every iteration set."""
    out = dict(base)
    for lp in loops:
        s = lp["iter"]
        if s in out:
            continue
        ind = [a for a in lp["args"] if a[0] == "indirect"]
        if ind:
            _, _, tset, _col, table = ind[0]
            out[s] = out[tset][np.asarray(table)[:, 0]]
        else:
            out[s] = trivial(sizes[s], nranks)
    return out


def halos(loops, owner: dict, nranks: int):
    """Per set, per rank: (owned, exec, nonexec, imports{src: ids}, exports{dst: ids})."""
    touched = []
    for lp in loops:
        for s in [lp["iter"]] + [a[2] for a in lp["args"] if a[2] is not None]:
            if s not in touched:
                touched.append(s)
    exec_h = {s: [set() for _ in range(nranks)] for s in touched}
    for lp in loops:
        it = owner[lp["iter"]]
        for kind, mode, tset, col, _table in lp["args"]:
            if kind != "indirect" or mode not in ("WRITE", "RW", "INC"):
                continue
            tgt_owner = owner[tset][col]
            for e in range(len(it)):
                if tgt_owner[e] != it[e]:
                    exec_h[lp["iter"]][int(tgt_owner[e])].add(e)
    nonexec = {s: [set() for _ in range(nranks)] for s in touched}
    for lp in loops:
        s = lp["iter"]
        it = owner[s]
        for r in range(nranks):
            executed = [e for e in range(len(it)) if it[e] == r or e in exec_h[s][r]]
            for kind, _mode, tset, col, _table in lp["args"]:
                if kind != "indirect":
                    continue
                for e in executed:
                    t = int(col[e])
                    if owner[tset][t] != r and t not in exec_h[tset][r]:
                        nonexec[tset][r].add(t)
    result = {}
    for s in touched:
        per = []
        for r in range(nranks):
            owned = np.flatnonzero(owner[s] == r)
            ex = np.array(sorted(exec_h[s][r]), dtype=np.int64)
            nx = np.array(sorted(nonexec[s][r]), dtype=np.int64)
            halo = sorted(exec_h[s][r] | nonexec[s][r])
            imports = {}
            for g in halo:
                imports.setdefault(int(owner[s][g]), []).append(g)
            per.append([owned, ex, nx, {k: np.array(v, dtype=np.int64)
                                        for k, v in sorted(imports.items())}, {}])
        for r in range(nranks):
            for src, ids in per[r][3].items():
                per[src][4][r] = ids
        result[s] = per
    return result
