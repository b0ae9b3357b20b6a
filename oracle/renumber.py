"""Renumbering oracle (TEST ORACLE ONLY): Cuthill–McKee over map co-occurrence.

Restates reference ``renumber.py``:

* adjacency of a set S (53-81): every pair of columns (i < j) of every map
  whose *target* set is S contributes the pairs (t_i, t_j); self pairs are
  dropped, the graph is symmetrised and de-duplicated, neighbours of a
  vertex are ascending.  A set with no incident map (either direction) is
  an error;
* ordering (84-128): components in ascending order of their lowest vertex;
  each component restarts from its minimum-(degree, index) vertex; BFS
  appends unseen neighbours sorted by (degree, index).  NOT reversed — it
  is Cuthill–McKee although the package calls it RCM; ``forward[order] =
  arange``;
* source-set order (131-138): stable lexicographic sort of map rows,
  column 0 most significant;
* ``apply`` (141-166), ``span`` metric (169-174) and the driver order
  (177-202): target sets first in declaration order, then each remaining
  source set by its first declared map.

Operates on plain arrays: ``maps`` is a list of dicts
``{"name", "from", "to", "table"}`` in declaration order.
"""
from __future__ import annotations

from collections import deque

import numpy as np

__all__ = ["adjacency", "cm_order", "row_order", "span_stats", "renumber"]


def adjacency(maps, set_name: str, n: int):
    incident = [m for m in maps if m["to"] == set_name or m["from"] == set_name]
    if not incident:
        raise ValueError(f"set {set_name!r} has no incident map")
    nbrs = [set() for _ in range(n)]
    for m in incident:
        t = np.asarray(m["table"])
        if m["to"] != set_name or t.shape[0] == 0:
            continue
        for row in t.tolist():
            for i in range(len(row)):
                for j in range(i + 1, len(row)):
                    a, b = row[i], row[j]
                    if a != b:
                        nbrs[a].add(b)
                        nbrs[b].add(a)
    return [sorted(s) for s in nbrs]


def cm_order(nbrs) -> np.ndarray:
    n = len(nbrs)
    deg = [len(s) for s in nbrs]
    placed = [False] * n
    order = []
    for lead in range(n):
        if placed[lead]:
            continue
        # the whole component of `lead`
        comp, todo, inside = [], deque([lead]), {lead}
        while todo:
            v = todo.popleft()
            comp.append(v)
            for w in nbrs[v]:
                if w not in inside:
                    inside.add(w)
                    todo.append(w)
        start = min(comp, key=lambda v: (deg[v], v))
        seen = {start}
        frontier = deque([start])
        while frontier:
            v = frontier.popleft()
            order.append(v)
            placed[v] = True
            fresh = sorted((w for w in nbrs[v] if w not in seen), key=lambda w: (deg[w], w))
            seen.update(fresh)
            frontier.extend(fresh)
    return np.array(order, dtype=np.int64)


def forward_of(order: np.ndarray) -> np.ndarray:
    fwd = np.empty(order.size, dtype=np.int64)
    fwd[order] = np.arange(order.size)
    return fwd


def row_order(table) -> np.ndarray:
    t = np.asarray(table)
    rows = sorted(range(t.shape[0]), key=lambda r: tuple(t[r].tolist()))   # sorted() is stable
    return np.array(rows, dtype=np.int64)


def span_stats(table) -> tuple[int, float]:
    t = np.asarray(table)
    if t.shape[0] == 0:
        return 0, 0.0
    spans = [max(r) - min(r) for r in t.tolist()]
    return int(max(spans)), float(np.mean(spans))


def renumber(sets: dict, maps: list, dats: list):
    """Whole-mesh renumbering on arrays (renumber.py:177-202).

    ``sets`` name->size (declaration order), ``maps`` as above, ``dats`` a
    list of ``{"set", "values"}`` with logical ``(size, dim)`` values.
    Returns ``(forward per set, new maps, new dats)``.
    """
    maps = [dict(m, table=np.asarray(m["table"]).copy()) for m in maps]
    dats = [dict(d, values=np.asarray(d["values"]).copy()) for d in dats]
    fwds = {}

    def apply(sname, fwd):
        for d in dats:
            if d["set"] == sname:
                moved = np.empty_like(d["values"])
                moved[fwd] = d["values"]
                d["values"] = moved
        for m in maps:
            if m["to"] == sname:
                m["table"] = fwd[m["table"]]
            if m["from"] == sname:
                moved = np.empty_like(m["table"])
                moved[fwd] = m["table"]
                m["table"] = moved

    for s, size in sets.items():
        if any(m["to"] == s for m in maps):
            fwd = forward_of(cm_order(adjacency(maps, s, size)))
            apply(s, fwd)
            fwds[s] = fwd
    for s in sets:
        if s in fwds or not any(m["from"] == s for m in maps):
            continue
        primary = next(m for m in maps if m["from"] == s)
        fwd = forward_of(row_order(primary["table"]))
        apply(s, fwd)
        fwds[s] = fwd
    return fwds, maps, dats
