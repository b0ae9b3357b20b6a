"""Case builders shared by CPU and GPU tests (product API).

They rebuild, with :mod:`paper_1403_7209_b200`, the same meshes and loops
``tests/golden/make_golden.py`` built with the reference, and tag the
ad-hoc test kernels with the device functors that implement them.
"""
from __future__ import annotations

import numpy as np

import paper_1403_7209_b200 as ml
from paper_1403_7209_b200 import apps
from paper_1403_7209_b200.kernels import device_kernel


def _scatter_kernel(arity: int):
    @device_kernel(f"scatter_src_{arity}")
    def kern(s, *targets):
        for t in targets:
            t[0] += s[0]
    return kern


def _inc_kernel(arity: int):
    @device_kernel(f"inc_one_{arity}")
    def kern(*views):
        for v in views:
            v[0] += 1
    return kern


def _write_kernel(arity: int):
    @device_kernel(f"write_src_{arity}")
    def kern(s, *views):
        for k, v in enumerate(views):
            v[0] = s[0] + k
    return kern


def write_loop(mesh, map_name="m", src_name="src", dat_name="vals"):
    """Conflicting indirect WRITEs: serial order decides (last writer wins)."""
    m = mesh.maps[map_name]
    args = [ml.arg_direct(mesh.dats[src_name], ml.READ)] + [
        ml.arg_indirect(mesh.dats[dat_name], m, k + 1, ml.WRITE) for k in range(m.arity)]
    return ml.Loop("write_conflicts", m.from_set, args, _write_kernel(m.arity))


def random_loop_mesh(rng, max_elems=500):
    """reference tests/conftest.py:59-79, same RNG draw order."""
    nt = int(rng.integers(2, max(3, max_elems // 3)))
    ni = int(rng.integers(1, max(2, max_elems - nt)))
    arity = int(rng.integers(1, 4))
    mesh = ml.Mesh()
    tgt = mesh.decl_set("tgt", nt)
    it = mesh.decl_set("it", ni)
    m = mesh.decl_map("m", it, tgt, arity, rng.integers(1, nt + 1, size=ni * arity))
    vals = mesh.decl_dat("vals", tgt, 1, "int64", np.zeros(nt, dtype=np.int64))
    src = mesh.decl_dat("src", it, 1, "int64", rng.integers(0, 100, size=ni).astype(np.int64))
    args = [ml.arg_direct(src, ml.READ)] + [ml.arg_indirect(vals, m, k + 1, ml.INC)
                                            for k in range(arity)]
    return mesh, ml.Loop("fuzz", it, args, _scatter_kernel(arity))


def inc_loop(mesh, map_name="edge_nodes", dat_name="acc", dtype="int64"):
    """reference tests/conftest.py:43-56."""
    m = mesh.maps[map_name]
    if dat_name not in mesh.dats:
        mesh.decl_dat(dat_name, m.to_set, 1, dtype, np.zeros(m.to_set.size, dtype=dtype))
    dat = mesh.dats[dat_name]
    args = [ml.arg_indirect(dat, m, k + 1, ml.INC) for k in range(m.arity)]
    return ml.Loop(f"inc_{map_name}", m.from_set, args, _inc_kernel(m.arity))


def path_mesh(order=(1, 2, 3, 4)):
    mesh = ml.Mesh()
    nodes = mesh.decl_set("nodes", 4)
    edges = mesh.decl_set("edges", 3)
    rows = []
    for k in range(3):
        rows.extend((order[k], order[k + 1]))
    mesh.decl_map("edge_nodes", edges, nodes, 2, rows)
    return mesh


@device_kernel("mixmax")
def _k_mixmax(w1, w2, a1, a2, s, lo_, hi_):
    a1[:] += w2 * s[0]
    a2[:] += w1 * s[0]
    m, big = int(min(w1.min(), w2.min())), int(max(w1.max(), w2.max()))
    if m < lo_[0]:
        lo_[0] = m
    if big > hi_[0]:
        hi_[0] = big


def mixmax_case(auto_soa_threshold=4):
    """reference tests/test_executor.py:367-394."""
    mesh = ml.Mesh(auto_soa_threshold=auto_soa_threshold)
    nodes = mesh.decl_set("nodes", 30)
    edges = mesh.decl_set("edges", 60)
    rng = np.random.default_rng(7)
    en = mesh.decl_map("en", edges, nodes, 2, rng.integers(1, 31, 120))
    wide = mesh.decl_dat("wide", nodes, 5, "int64", rng.integers(-9, 9, 150))
    acc = mesh.decl_dat("acc", nodes, 5, "int64", np.zeros(150, np.int64))
    lo, hi, scale = ml.Global(np.int64(10 ** 9)), ml.Global(np.int64(-10 ** 9)), ml.Global(np.int64(3))
    loop = ml.Loop("mixmax", edges, [
        ml.arg_indirect(wide, en, 1, ml.READ), ml.arg_indirect(wide, en, 2, ml.READ),
        ml.arg_indirect(acc, en, 1, ml.INC), ml.arg_indirect(acc, en, 2, ml.INC),
        ml.arg_global(scale, ml.READ), ml.arg_global(lo, ml.MIN), ml.arg_global(hi, ml.MAX),
    ], _k_mixmax)
    return mesh, loop, acc, lo, hi


def build_app(app: str, n: int, dtype: str, steps: int):
    """The reference app programs, built with the product API."""
    mesh = apps.sample_mesh() if n == 0 else apps.gen_mesh(n)
    if app == "diffusion":
        prog, h = apps.build_diffusion(mesh, steps, dtype=dtype)
    else:
        prog, h = apps.build_cell_area(mesh, dtype)
    return mesh, prog, h


def app_results(app: str, h) -> dict:
    if app == "diffusion":
        return {"u": h["u"].fetch(), "flux": h["flux"].fetch(),
                "residuals": np.array([g.value for g in h["residuals"]])}
    return {"arean": h["arean"].fetch(), "areac": h["areac"].fetch(),
            "total": np.atleast_1d(h["total"].value)}
