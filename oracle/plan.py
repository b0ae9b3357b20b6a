"""Execution-plan oracle: blocks + two-level greedy colouring (TEST ORACLE ONLY).

Restates ``build_plan`` (reference ``plan.py:55-131``) with a different
formulation that yields the same arrays:

* blocks are contiguous ``block_size`` ranges, the last ragged (64-66);
* write targets are ``(dat key, map column)`` pairs, made disjoint across
  dats by per-key offsets.  QUIRK kept on purpose (plan.py:77-81): a key's
  offset width is ``max(first column seen for that key) + 1``, so a later
  column of the same dat with larger ids can alias into the next key's
  range and create false (safe) conflicts;
* block colour = smallest colour not used by any *lower-index* block that
  shares a write target (plan.py:82-103).  Scanning blocks in index order and
  remembering, per target, the set of colours of blocks already coloured
  that touch it gives exactly that set;
* element colour, per block, in element order, over all of the element's
  targets (plan.py:105-123);
* ``block_elem_order[b]`` = block elements stably sorted by element colour
  (plan.py:126-129); no indirect writes -> one colour (70-72); empty -> 0.

Pure Python over bitsets: fine for the small/medium cases tests use.
"""
from __future__ import annotations

from dataclasses import dataclass

import numpy as np

__all__ = ["OraclePlan", "build_plan", "write_columns", "race_free"]


@dataclass
class OraclePlan:
    n: int
    block_size: int
    nblocks: int
    block_bounds: np.ndarray
    block_color: np.ndarray
    ncolors: int
    blocks_by_color: list
    elem_color: np.ndarray
    elem_ncolors: np.ndarray
    block_elem_order: list


def write_columns(loop) -> list:
    """``(dat name, target column)`` per indirect WRITE/RW/INC argument (plan.py:134-135)."""
    return [(a.dat.name, np.asarray(a.map.table[:, a.slot]))
            for a in loop.args
            if a.kind == "indirect" and a.mode.name in ("WRITE", "RW", "INC")]


def _lowest_free(mask: int) -> int:
    return ((~mask) & (mask + 1)).bit_length() - 1


def build_plan(n: int, write_cols, block_size: int) -> OraclePlan:
    if block_size < 1:
        raise ValueError(f"block size must be >= 1, got {block_size}")
    nb = (n + block_size - 1) // block_size
    bounds = np.array([min(i * block_size, n) for i in range(nb + 1)], dtype=np.int64)
    elem_color = np.zeros(n, dtype=np.int64)
    elem_nc = np.ones(nb, dtype=np.int64)
    block_color = np.zeros(nb, dtype=np.int64)

    if write_cols and n:
        width, base = {}, {}
        for key, col in write_cols:
            if key not in base:
                base[key] = sum(width.values())
                width[key] = int(np.max(col)) + 1 if len(col) else 0
        targets = np.stack([np.asarray(col, dtype=np.int64) + base[key]
                            for key, col in write_cols], axis=1)     # (n, ncols)
        rows = targets.tolist()
        # block level: per target, bitset of colours of already-coloured blocks
        used_at: dict[int, int] = {}
        for b in range(nb):
            lo, hi = int(bounds[b]), int(bounds[b + 1])
            mine = {t for r in rows[lo:hi] for t in r}
            forbid = 0
            for t in mine:
                forbid |= used_at.get(t, 0)
            c = _lowest_free(forbid)
            block_color[b] = c
            for t in mine:
                used_at[t] = used_at.get(t, 0) | (1 << c)
        # element level, independently per block
        for b in range(nb):
            lo, hi = int(bounds[b]), int(bounds[b + 1])
            local: dict[int, int] = {}
            top = 0
            for e in range(lo, hi):
                forbid = 0
                for t in rows[e]:
                    forbid |= local.get(t, 0)
                c = _lowest_free(forbid)
                elem_color[e] = c
                top = max(top, c)
                for t in rows[e]:
                    local[t] = local.get(t, 0) | (1 << c)
            elem_nc[b] = top + 1
        ncolors = int(block_color.max()) + 1 if nb else 0
    else:
        ncolors = 1 if nb else 0

    by_color = [np.flatnonzero(block_color == c) for c in range(ncolors)]
    order = [int(bounds[b]) + np.argsort(elem_color[bounds[b]:bounds[b + 1]], kind="stable")
             for b in range(nb)]
    return OraclePlan(n, block_size, nb, bounds, block_color, ncolors, by_color,
                      elem_color, elem_nc, order)


def race_free(plan, write_targets_of) -> bool:
    """Exhaustive scan: no two same-colour blocks (or same-colour elements in a
    block) share a write target.  ``write_targets_of(e)`` -> set of targets.
    Mirrors the independent oracle of reference tests/conftest.py:137-160."""
    per_block = []
    for b in range(plan.nblocks):
        s = set()
        for e in range(int(plan.block_bounds[b]), int(plan.block_bounds[b + 1])):
            s |= write_targets_of(e)
        per_block.append(s)
    for c in range(plan.ncolors):
        seen = set()
        for b in plan.blocks_by_color[c]:
            if seen & per_block[int(b)]:
                return False
            seen |= per_block[int(b)]
    for b in range(plan.nblocks):
        lo, hi = int(plan.block_bounds[b]), int(plan.block_bounds[b + 1])
        for c in range(int(plan.elem_ncolors[b])):
            seen = set()
            for e in range(lo, hi):
                if plan.elem_color[e] == c:
                    t = write_targets_of(e)
                    if seen & t:
                        return False
                    seen |= t
    return True
