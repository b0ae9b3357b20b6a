"""Bundled solver programs and synthetic mesh generators.

Programs (same loop rosters as the reference ``pkg/src/meshloop/apps.py``):

* :func:`build_cell_area` — triangle areas, scatter a third to each node,
  global total (reference apps.py:159-201);
* :func:`build_diffusion` — explicit graph-Laplacian relaxation, one
  residual reduction per step; ``edge_flux`` is the indirect-INC hot loop
  (reference apps.py:228-304);
* :func:`build_hydra_proxy` — NEW: a Hydra-shaped iteration (paper Table 2,
  ``PAPER.md:766-779``) with wide SOA dats, three indirect edge loops
  (``grad_edge``, ``iflux`` 34/12 doubles, ``vflux`` 92/12 doubles), a MIN
  local-timestep reduction feeding a READ global, a SUM residual and an
  indirect boundary write.  It is the benchmark workload.

Generators: :func:`gen_mesh` (2-D triangulated square, restated from
reference apps.py:49-105 so numbering is identical), :func:`sample_mesh`
(the paper's Fig. 2 disk), :func:`gen_hex_mesh` / :func:`gen_kuhn_mesh`
(3-D grids with jittered coordinates), :func:`shuffle_mesh` (random
renumbering, makes a structured mesh "unstructured") and
:func:`gen_hub_mesh` (colouring stress: hub nodes of very high degree).

Every Python kernel here is tagged with the device functor that implements
it on the GPU; the Python body is the per-element semantics the test oracle
executes.
"""
from __future__ import annotations

import math

import numpy as np

from .core import (INC, MIN, READ, RW, WRITE, ExecError, Global, Loop, Mesh,
                   arg_direct, arg_global, arg_indirect)
from .kernels import device_kernel

__all__ = [
    "gen_mesh", "sample_mesh", "gen_hex_mesh", "gen_kuhn_mesh", "gen_hub_mesh",
    "shuffle_mesh", "build_cell_area", "build_diffusion", "build_hydra_proxy",
    "UnstableTimestep", "stability_bound", "check_residual_history",
]


class UnstableTimestep(ExecError):
    """Explicit diffusion step exceeds the stable timestep bound."""


def _require(mesh: Mesh, sets=(), maps=(), dats=()):
    missing = ([f"set {n!r}" for n in sets if n not in mesh.sets]
               + [f"map {n!r}" for n in maps if n not in mesh.maps]
               + [f"dat {n!r}" for n in dats if n not in mesh.dats])
    if missing:
        raise ExecError("mesh lacks required " + ", ".join(missing))


# -- generators ----------------------------------------------------------------

def gen_mesh(n: int, auto_soa_threshold: int | None = 4) -> Mesh:
    """Triangulated unit square: (n+1)^2 nodes, 2n^2 cells, 3n^2+2n edges, 4n bedges.

    Numbering identical to reference apps.py:49-105: nodes row-major; cells
    split along the (ix,iy)->(ix+1,iy+1) diagonal; edges horizontals, then
    verticals, then diagonals; boundary edges bottom, top, left, right.
    """
    if n < 1:
        raise ValueError(f"refinement must be >= 1, got {n}")
    mesh = Mesh(auto_soa_threshold=auto_soa_threshold)
    w = n + 1
    nodes = mesh.decl_set("nodes", w * w)
    edges = mesh.decl_set("edges", 3 * n * n + 2 * n)
    cells = mesh.decl_set("cells", 2 * n * n)
    bedges = mesh.decl_set("bedges", 4 * n)

    iy, ix = np.meshgrid(np.arange(n), np.arange(n), indexing="ij")
    a = (iy * w + ix + 1).ravel()          # 1-based ids of the square's corners
    b, c, d = a + 1, a + w + 1, a + w
    cell_rows = np.stack([np.stack([a, b, c], 1), np.stack([a, c, d], 1)], 1).reshape(-1, 3)

    hy, hx = np.meshgrid(np.arange(w), np.arange(n), indexing="ij")
    horiz = (hy * w + hx + 1).ravel()
    vy, vx = np.meshgrid(np.arange(n), np.arange(w), indexing="ij")
    vert = (vy * w + vx + 1).ravel()
    edge_rows = np.concatenate([np.stack([horiz, horiz + 1], 1),
                                np.stack([vert, vert + w], 1),
                                np.stack([a, a + w + 1], 1)])
    k = np.arange(n)
    bottom, top = k + 1, n * w + k + 1
    left, right = k * w + 1, k * w + n + 1
    bedge_rows = np.concatenate([np.stack([bottom, bottom + 1], 1), np.stack([top, top + 1], 1),
                                 np.stack([left, left + w], 1), np.stack([right, right + w], 1)])

    mesh.decl_map("cell_nodes", cells, nodes, 3, cell_rows.ravel())
    mesh.decl_map("edge_nodes", edges, nodes, 2, edge_rows.ravel())
    mesh.decl_map("bedge_nodes", bedges, nodes, 2, bedge_rows.ravel())
    gy, gx = np.meshgrid(np.arange(w), np.arange(w), indexing="ij")
    coords = np.stack([gx.ravel() / n, gy.ravel() / n], 1)
    mesh.decl_dat("coords", nodes, 2, "float64", coords.ravel())
    return mesh


_FIG2_CELLS = np.array([
    (1, 3, 10), (1, 2, 3), (3, 9, 10), (2, 3, 4), (3, 4, 9),
    (9, 14, 10), (14, 13, 10), (13, 12, 10), (12, 1, 10), (12, 11, 1),
    (11, 8, 1), (8, 2, 1), (8, 7, 2), (7, 4, 2), (7, 6, 4),
    (6, 5, 4), (5, 9, 4)])
_FIG2_COORDS = np.array([
    (-0.6, 0.8), (0.6, 0.8), (0.0, 0.0), (1.0, -0.3), (0.9, -1.6),
    (1.8, -1.2), (2.2, 0.2), (1.2, 1.6), (0.0, -1.1), (-1.0, -0.3),
    (0.0, 2.1), (-1.2, 1.6), (-2.2, 0.2), (-1.8, -1.2)])


def sample_mesh(auto_soa_threshold: int | None = 4) -> Mesh:
    """The paper's Fig. 2 disk: 14 nodes, 17 cells (reference apps.py:108-131)."""
    mesh = Mesh(auto_soa_threshold=auto_soa_threshold)
    nodes = mesh.decl_set("nodes", 14)
    cells = mesh.decl_set("cells", 17)
    mesh.decl_map("cell_nodes", cells, nodes, 3, _FIG2_CELLS.ravel())
    mesh.decl_dat("coords", nodes, 2, "float64", _FIG2_COORDS.ravel())
    return mesh


def _grid_ids(N: int) -> np.ndarray:
    """1-based node ids of an N^3 grid indexed [z, y, x] (x fastest)."""
    return np.arange(1, N ** 3 + 1, dtype=np.int64).reshape(N, N, N)


def _axis_edges(ids: np.ndarray) -> list[np.ndarray]:
    """Axis-aligned node pairs (x, then y, then z direction)."""
    return [np.stack([ids[:, :, :-1].ravel(), ids[:, :, 1:].ravel()], 1),
            np.stack([ids[:, :-1, :].ravel(), ids[:, 1:, :].ravel()], 1),
            np.stack([ids[:-1, :, :].ravel(), ids[1:, :, :].ravel()], 1)]


def _grid_mesh(N: int, rows: np.ndarray, seed: int, jitter: float,
               auto_soa_threshold) -> Mesh:
    ids = _grid_ids(N)
    on_surface = np.zeros((N, N, N), dtype=bool)
    on_surface[[0, -1], :, :] = on_surface[:, [0, -1], :] = on_surface[:, :, [0, -1]] = True
    surf = on_surface.ravel()
    brows = rows[surf[rows[:, 0] - 1] & surf[rows[:, 1] - 1]]
    mesh = Mesh(auto_soa_threshold=auto_soa_threshold)
    nodes = mesh.decl_set("nodes", N ** 3)
    edges = mesh.decl_set("edges", len(rows))
    bedges = mesh.decl_set("bedges", len(brows))
    mesh.decl_map("edge_nodes", edges, nodes, 2, rows.ravel())
    mesh.decl_map("bedge_nodes", bedges, nodes, 2, brows.ravel())
    h = 1.0 / max(N - 1, 1)
    z, y, x = np.meshgrid(np.arange(N), np.arange(N), np.arange(N), indexing="ij")
    xyz = np.stack([x.ravel(), y.ravel(), z.ravel()], 1) * h
    rng = np.random.default_rng(seed)
    xyz = xyz + rng.uniform(-jitter * h, jitter * h, size=xyz.shape)
    mesh.decl_dat("coords", nodes, 3, "float64", xyz.ravel())
    return mesh


def gen_hex_mesh(N: int, seed: int = 0, jitter: float = 0.25,
                 auto_soa_threshold: int | None = 4) -> Mesh:
    """3-D grid graph: N^3 nodes, 3 N^2 (N-1) axis edges, boundary-surface bedges.

    N=94 gives 830,584 nodes / 2,465,244 edges (Rotor37-sized),
    N=139 gives 2,685,619 / 7,998,894 (the 8M-edge multi-GPU mesh).
    Coordinates are jittered by ±``jitter``·h (seeded) so RCB sees an
    unstructured point cloud.
    """
    if N < 2:
        raise ValueError(f"grid needs N >= 2, got {N}")
    rows = np.concatenate(_axis_edges(_grid_ids(N)))
    return _grid_mesh(N, rows, seed, jitter, auto_soa_threshold)


def gen_kuhn_mesh(N: int, seed: int = 0, jitter: float = 0.25,
                  auto_soa_threshold: int | None = 4) -> Mesh:
    """3-D Kuhn (6-tet) split of an N^3 grid: axis + face + body diagonals.

    N=47 gives 103,823 nodes / 700,534 edges (config 1 of BASELINE.json).
    """
    if N < 2:
        raise ValueError(f"grid needs N >= 2, got {N}")
    ids = _grid_ids(N)
    diag = [np.stack([ids[:, :-1, :-1].ravel(), ids[:, 1:, 1:].ravel()], 1),   # xy faces
            np.stack([ids[:-1, :, :-1].ravel(), ids[1:, :, 1:].ravel()], 1),   # xz faces
            np.stack([ids[:-1, :-1, :].ravel(), ids[1:, 1:, :].ravel()], 1),   # yz faces
            np.stack([ids[:-1, :-1, :-1].ravel(), ids[1:, 1:, 1:].ravel()], 1)]
    rows = np.concatenate(_axis_edges(ids) + diag)
    return _grid_mesh(N, rows, seed, jitter, auto_soa_threshold)


def gen_hub_mesh(n_nodes: int, n_edges: int, n_hubs: int = 8, hub_share: float = 0.02,
                 seed: int = 0, auto_soa_threshold: int | None = 4) -> Mesh:
    """Colouring stress mesh: random arity-2 edges, a few hubs of very high degree.

    A fraction ``hub_share`` of the edges has one end on one of ``n_hubs``
    hub nodes (degree ~ hub_share*n_edges/n_hubs); the rest join uniformly
    random node pairs, in the style of the reference fuzz meshes
    (tests/conftest.py:59-79).
    """
    rng = np.random.default_rng(seed)
    ends = rng.integers(1, n_nodes + 1, size=(n_edges, 2))
    hubbed = rng.random(n_edges) < hub_share
    ends[hubbed, 0] = rng.integers(1, n_hubs + 1, size=int(hubbed.sum()))
    same = ends[:, 0] == ends[:, 1]
    ends[same, 1] = ends[same, 1] % n_nodes + 1
    mesh = Mesh(auto_soa_threshold=auto_soa_threshold)
    nodes = mesh.decl_set("nodes", n_nodes)
    edges = mesh.decl_set("edges", n_edges)
    bedges = mesh.decl_set("bedges", 0)
    mesh.decl_map("edge_nodes", edges, nodes, 2, ends.ravel())
    mesh.decl_map("bedge_nodes", bedges, nodes, 2, np.empty(0, np.int64))
    mesh.decl_dat("coords", nodes, 3, "float64", rng.random(3 * n_nodes))
    return mesh


def shuffle_mesh(mesh: Mesh, seed: int = 0, sets=None) -> dict:
    """Randomly renumber ``sets`` (default: every set) in place; returns the permutations.

    Uses :func:`paper_1403_7209_b200.renumber.apply_permutation`, so it must
    run before the mesh freezes.
    """
    from .renumber import Permutation, apply_permutation
    rng = np.random.default_rng(seed)
    out = {}
    for name in (sets or list(mesh.sets)):
        size = mesh.sets[name].size
        fwd = rng.permutation(size).astype(np.int64)
        perm = Permutation(name, fwd, np.argsort(fwd), mesh.version)
        apply_permutation(mesh, perm)
        out[name] = perm
    return out


# -- cell-area app (reference apps.py:134-201) --------------------------------------

@device_kernel("tri_area")
def _k_tri_area(c1, c2, c3, out):
    out[0] = 0.5 * abs((c2[0] - c1[0]) * (c3[1] - c1[1]) - (c3[0] - c1[0]) * (c2[1] - c1[1]))


@device_kernel("distribute")
def _k_distribute(ac, a1, a2, a3):
    third = ac[0] / 3.0
    a1[0] += third
    a2[0] += third
    a3[0] += third


@device_kernel("distribute_int")
def _k_distribute_int(ac, a1, a2, a3):
    third = ac[0] // 3
    a1[0] += third
    a2[0] += third
    a3[0] += third


@device_kernel("sum")
def _k_sum(v, total):
    total[0] += v[0]


def build_cell_area(mesh: Mesh, dtype: str = "float64"):
    """Per-node area shares and their total; int64 twin seeds cell areas 3,6,9,..."""
    _require(mesh, sets=("cells", "nodes"), maps=("cell_nodes",),
             dats=("coords",) if dtype == "float64" else ())
    cells, nodes = mesh.sets["cells"], mesh.sets["nodes"]
    cn = mesh.maps["cell_nodes"]
    program = []
    if dtype == "float64":
        areac = mesh.decl_dat("areac", cells, 1, dtype, np.zeros(cells.size))
        arean = mesh.decl_dat("arean", nodes, 1, dtype, np.zeros(nodes.size))
        total = Global(np.zeros(1), name="area_total")
        coords = mesh.dats["coords"]
        program.append(Loop("area_calc", cells, [
            arg_indirect(coords, cn, 1, READ), arg_indirect(coords, cn, 2, READ),
            arg_indirect(coords, cn, 3, READ), arg_direct(areac, WRITE)], _k_tri_area))
        distribute = _k_distribute
    else:
        areac = mesh.decl_dat("areac", cells, 1, dtype,
                              3 * np.arange(1, cells.size + 1, dtype=np.int64))
        arean = mesh.decl_dat("arean", nodes, 1, dtype, np.zeros(nodes.size, dtype=np.int64))
        total = Global(np.zeros(1, dtype=np.int64), name="area_total")
        distribute = _k_distribute_int
    program.append(Loop("area_distribute", cells, [
        arg_direct(areac, READ), arg_indirect(arean, cn, 1, INC),
        arg_indirect(arean, cn, 2, INC), arg_indirect(arean, cn, 3, INC)], distribute))
    program.append(Loop("area_total", nodes, [arg_direct(arean, READ), arg_global(total, INC)],
                        _k_sum))
    return program, {"areac": areac, "arean": arean, "total": total}


# -- diffusion app (reference apps.py:204-316) ----------------------------------

def stability_bound(mesh: Mesh) -> float:
    """Largest stable explicit timestep: 1 / max node degree (unit weights)."""
    deg = np.bincount(mesh.maps["edge_nodes"].table.ravel(), minlength=mesh.sets["nodes"].size)
    return 1.0 / max(int(deg.max()), 1)


@device_kernel("copy")
def _k_copy(src, dst):
    dst[0] = src[0]


@device_kernel("edge_flux")
def _k_edge_flux(u1, u2, f1, f2):
    d = u2[0] - u1[0]
    f1[0] += d
    f2[0] -= d


@device_kernel("boundary_fix")
def _k_boundary_fix(u1, u2, g1, g2):
    u1[0] = g1[0]
    u2[0] = g2[0]


def build_diffusion(mesh: Mesh, steps: int, dt: float | None = None, dtype: str = "float64"):
    """``steps`` explicit diffusion steps: save, edge flux, node update (+residual), boundary."""
    _require(mesh, sets=("nodes", "edges", "bedges"), maps=("edge_nodes", "bedge_nodes"),
             dats=("coords",) if dtype == "float64" else ())
    nodes, edges, bedges = (mesh.sets[k] for k in ("nodes", "edges", "bedges"))
    en, bn = mesh.maps["edge_nodes"], mesh.maps["bedge_nodes"]
    bound = stability_bound(mesh)
    if dtype == "float64":
        if dt is None:
            dt = 0.9 * bound
        if dt > bound * (1 + 1e-12):
            raise UnstableTimestep(f"dt={dt} exceeds the stable bound 1/max_degree = {bound}")
        x = mesh.dats["coords"].fetch()[:, 0]
        u = mesh.decl_dat("u", nodes, 1, dtype, np.zeros(nodes.size))
        u0 = mesh.decl_dat("u_prev", nodes, 1, dtype, np.zeros(nodes.size))
        flux = mesh.decl_dat("flux", nodes, 1, dtype, np.zeros(nodes.size))
        g = mesh.decl_dat("bc_values", nodes, 1, dtype, x)

        @device_kernel("diffusion_update", consts="float_defaults")
        def _k_update(u_, up, f, res, dt=float(dt)):
            nu = up[0] + dt * f[0]
            res[0] += f[0] * f[0]
            u_[0] = nu
            f[0] = 0.0
        res_dtype = np.float64
    else:
        scale = int(round(1.0 / bound)) + 1
        ids = np.arange(nodes.size, dtype=np.int64)
        u = mesh.decl_dat("u", nodes, 1, dtype, (ids * 7) % 23)
        u0 = mesh.decl_dat("u_prev", nodes, 1, dtype, np.zeros(nodes.size, np.int64))
        flux = mesh.decl_dat("flux", nodes, 1, dtype, np.zeros(nodes.size, np.int64))
        g = mesh.decl_dat("bc_values", nodes, 1, dtype, (ids * 13) % 31)

        @device_kernel("diffusion_update", consts="int_defaults")
        def _k_update(u_, up, f, res, scale=scale):
            nu = up[0] + f[0] // scale
            res[0] += abs(f[0])
            u_[0] = nu
            f[0] = 0
        res_dtype = np.int64

    residuals = [Global(np.zeros(1, dtype=res_dtype), name=f"residual_{k}") for k in range(steps)]
    program = []
    for k in range(steps):
        program += [
            Loop("state_save", nodes, [arg_direct(u, READ), arg_direct(u0, WRITE)], _k_copy),
            Loop("edge_flux", edges, [arg_indirect(u, en, 1, READ), arg_indirect(u, en, 2, READ),
                                      arg_indirect(flux, en, 1, INC),
                                      arg_indirect(flux, en, 2, INC)], _k_edge_flux),
            Loop("node_update", nodes, [arg_direct(u, WRITE), arg_direct(u0, READ),
                                        arg_direct(flux, RW), arg_global(residuals[k], INC)],
                 _k_update),
            Loop("boundary_fix", bedges, [arg_indirect(u, bn, 1, WRITE),
                                          arg_indirect(u, bn, 2, WRITE),
                                          arg_indirect(g, bn, 1, READ),
                                          arg_indirect(g, bn, 2, READ)], _k_boundary_fix),
        ]
    handles = {"u": u, "flux": flux, "bc_values": g, "residuals": residuals,
               "dt": dt, "dt_bound": bound}
    return program, handles


def check_residual_history(residuals) -> np.ndarray:
    """Flag sustained residual growth (an unstable timestep) after a run."""
    hist = np.array([r.value for r in residuals], dtype=np.float64)
    if hist.size >= 4:
        ref = max(hist[:3].max(), np.finfo(np.float64).tiny)
        if hist[-1] > 10.0 * ref and np.all(np.diff(hist[-3:]) > 0):
            raise UnstableTimestep(f"residual history grows (last={hist[-1]:.3e}); "
                                   f"timestep exceeds the stable bound")
    return hist


# -- Hydra-shaped proxy iteration (benchmark workload) -----------------------------
#
# Shapes follow the paper's per-loop data table:
#   ifluxedge  direct 3/0, indirect 34/12 doubles  ->  iflux below
#   vfluxedge  direct 3/0, indirect 92/12 doubles  ->  vflux below
# The arithmetic is a stable, diffusive stand-in (Hydra's RANS physics is
# proprietary and out of scope); every value a loop reads influences what it
# writes, so no load can be dead-code-eliminated on the device.

NQ = 6          # flow variables per node (rho, rho*u, rho*v, rho*w, rho*E, nu~)
NG = 3 * NQ     # gradient components
NLIM = 8        # limiter data
NAUX = 19       # viscous / turbulence auxiliaries


@device_kernel("proxy_save")
def _k_proxy_save(q, q_old):
    for v in range(NQ):
        q_old[v] = q[v]


@device_kernel("proxy_dt", consts="float_defaults")
def _k_proxy_dt(q, vol, dt_loc, dt_min, cfl=0.05):
    s = 1.0
    for v in range(NQ):
        s = s + abs(q[v])
    d = cfl * vol[0] / s
    dt_loc[0] = d
    if d < dt_min[0]:
        dt_min[0] = d


@device_kernel("proxy_grad")
def _k_proxy_grad(w, q1, q2, x1, x2, g1, g2):
    for v in range(NQ):
        qa = 0.5 * (q1[v] + q2[v])
        dq = q2[v] - q1[v]
        for k in range(3):
            f = qa * w[k] + 0.125 * dq * (x2[k] - x1[k])
            g1[3 * v + k] += f
            g2[3 * v + k] -= f


@device_kernel("proxy_iflux")
def _k_proxy_iflux(w, q1, q2, x1, x2, l1, l2, r1, r2):
    d0, d1, d2 = x2[0] - x1[0], x2[1] - x1[1], x2[2] - x1[2]
    ds = math.sqrt(d0 * d0 + d1 * d1 + d2 * d2)
    an = math.sqrt(w[0] * w[0] + w[1] * w[1] + w[2] * w[2])
    s = 0.0
    for j in range(NLIM):
        t = l1[j] + l2[j]
        s = s + t * t
    lam = an / ((1.0 + ds) * (1.0 + 0.0625 * s))
    for v in range(NQ):
        f = lam * (q2[v] - q1[v])
        r1[v] += f
        r2[v] -= f


@device_kernel("proxy_vflux")
def _k_proxy_vflux(w, q1, q2, g1, g2, x1, x2, a1, a2, r1, r2):
    d0, d1, d2 = x2[0] - x1[0], x2[1] - x1[1], x2[2] - x1[2]
    ds2 = d0 * d0 + d1 * d1 + d2 * d2 + 1e-12
    wd = w[0] * d0 + w[1] * d1 + w[2] * d2
    mu = 0.0
    for j in range(NAUX):
        mu = mu + (a1[j] + a2[j])
    mu = 0.01 * mu / (2.0 * NAUX)
    for v in range(NQ):
        b = 3 * v
        gx = 0.5 * (g1[b] + g2[b])
        gy = 0.5 * (g1[b + 1] + g2[b + 1])
        gz = 0.5 * (g1[b + 2] + g2[b + 2])
        dq = q2[v] - q1[v]
        corr = (dq - (gx * d0 + gy * d1 + gz * d2)) / ds2
        f = mu * (0.001 * (gx * w[0] + gy * w[1] + gz * w[2]) + corr * abs(wd))
        r1[v] += f
        r2[v] -= f


@device_kernel("proxy_update")
def _k_proxy_update(q, q_old, res, vol, grad, dt_min, rms):
    s = dt_min[0] / vol[0]
    for v in range(NQ):
        r = res[v]
        q[v] = q_old[v] + s * r
        rms[0] += r * r
        res[v] = 0.0
    for k in range(NG):
        grad[k] = 0.0


@device_kernel("proxy_bc")
def _k_proxy_bc(q1, q2, b1, b2):
    for v in range(NQ):
        q1[v] = b1[v]
        q2[v] = b2[v]


def build_hydra_proxy(mesh: Mesh, steps: int = 1, seed: int = 0, cfl: float = 0.05, api=None):
    """Hydra-shaped solver iteration repeated ``steps`` times (the benchmark program).

    Per iteration: ``save`` (q→q_old) → ``dt_calc`` (local dt + global MIN)
    → ``grad_edge`` (indirect INC dim 18) → ``iflux`` (34/12) → ``vflux``
    (92/12) → ``update`` (reads the MIN as a READ global, SUM residual,
    zeroes res/grad) → ``bc`` (indirect WRITE on boundary edges).
    Returns ``(program, handles)``.  ``api``: the package whose ``Global``,
    ``Loop``, ``arg_*`` and access modes build the program (default this one;
    the reference ``meshloop`` module builds it from reference objects, for
    the stock reference's own executors and the reference-object path).
    """
    _require(mesh, sets=("nodes", "edges", "bedges"), maps=("edge_nodes", "bedge_nodes"),
             dats=("coords",))
    if api is not None:
        Global, Loop = api.Global, api.Loop
        arg_direct, arg_indirect, arg_global = api.arg_direct, api.arg_indirect, api.arg_global
        READ, WRITE, RW, INC, MIN = api.READ, api.WRITE, api.RW, api.INC, api.MIN
    else:
        from .core import Global, Loop, arg_direct, arg_indirect, arg_global, READ, WRITE, RW, INC, MIN
    nodes, edges, bedges = (mesh.sets[k] for k in ("nodes", "edges", "bedges"))
    en, bn = mesh.maps["edge_nodes"], mesh.maps["bedge_nodes"]
    n, m = nodes.size, edges.size
    rng = np.random.default_rng(seed)
    xyz = mesh.dats["coords"].fetch()
    if xyz.shape[1] < 3:
        xyz = np.concatenate([xyz, np.zeros((n, 3 - xyz.shape[1]))], 1)
    x = mesh.decl_dat("x", nodes, 3, "float64", xyz.ravel())
    q0 = 1.0 + 0.5 * np.sin(3.0 * xyz[:, :1] + np.arange(NQ)[None, :]) * np.cos(2.0 * xyz[:, 1:2])
    q = mesh.decl_dat("q", nodes, NQ, "float64", q0.ravel())
    q_old = mesh.decl_dat("q_old", nodes, NQ, "float64", np.zeros(n * NQ))
    grad = mesh.decl_dat("grad", nodes, NG, "float64", np.zeros(n * NG))
    lim = mesh.decl_dat("lim", nodes, NLIM, "float64", rng.random(n * NLIM))
    aux = mesh.decl_dat("aux", nodes, NAUX, "float64", rng.random(n * NAUX))
    res = mesh.decl_dat("res", nodes, NQ, "float64", np.zeros(n * NQ))
    vol = mesh.decl_dat("vol", nodes, 1, "float64", 1.0 + rng.random(n))
    dt_loc = mesh.decl_dat("dt_loc", nodes, 1, "float64", np.zeros(n))
    q_bc = mesh.decl_dat("q_bc", nodes, NQ, "float64", q0.ravel())
    w = mesh.decl_dat("w", edges, 3, "float64", rng.uniform(-1.0, 1.0, 3 * m))

    @device_kernel("proxy_dt", consts="float_defaults")
    def _k_dt(q, vol, dt_loc, dt_min, cfl=float(cfl)):
        _k_proxy_dt(q, vol, dt_loc, dt_min, cfl)

    dt_mins = [Global(np.array([np.inf]), name=f"dt_min_{k}") for k in range(steps)]
    rmss = [Global(np.zeros(1), name=f"rms_{k}") for k in range(steps)]
    program = []
    for k in range(steps):
        program += [
            Loop("save", nodes, [arg_direct(q, READ), arg_direct(q_old, WRITE)], _k_proxy_save),
            Loop("dt_calc", nodes, [arg_direct(q, READ), arg_direct(vol, READ),
                                    arg_direct(dt_loc, WRITE), arg_global(dt_mins[k], MIN)], _k_dt),
            Loop("grad_edge", edges, [arg_direct(w, READ),
                                      arg_indirect(q, en, 1, READ), arg_indirect(q, en, 2, READ),
                                      arg_indirect(x, en, 1, READ), arg_indirect(x, en, 2, READ),
                                      arg_indirect(grad, en, 1, INC),
                                      arg_indirect(grad, en, 2, INC)], _k_proxy_grad),
            Loop("iflux", edges, [arg_direct(w, READ),
                                  arg_indirect(q, en, 1, READ), arg_indirect(q, en, 2, READ),
                                  arg_indirect(x, en, 1, READ), arg_indirect(x, en, 2, READ),
                                  arg_indirect(lim, en, 1, READ), arg_indirect(lim, en, 2, READ),
                                  arg_indirect(res, en, 1, INC), arg_indirect(res, en, 2, INC)],
                 _k_proxy_iflux),
            Loop("vflux", edges, [arg_direct(w, READ),
                                  arg_indirect(q, en, 1, READ), arg_indirect(q, en, 2, READ),
                                  arg_indirect(grad, en, 1, READ), arg_indirect(grad, en, 2, READ),
                                  arg_indirect(x, en, 1, READ), arg_indirect(x, en, 2, READ),
                                  arg_indirect(aux, en, 1, READ), arg_indirect(aux, en, 2, READ),
                                  arg_indirect(res, en, 1, INC), arg_indirect(res, en, 2, INC)],
                 _k_proxy_vflux),
            Loop("update", nodes, [arg_direct(q, WRITE), arg_direct(q_old, READ),
                                   arg_direct(res, RW), arg_direct(vol, READ),
                                   arg_direct(grad, WRITE), arg_global(dt_mins[k], READ),
                                   arg_global(rmss[k], INC)], _k_proxy_update),
            Loop("bc", bedges, [arg_indirect(q, bn, 1, WRITE), arg_indirect(q, bn, 2, WRITE),
                                arg_indirect(q_bc, bn, 1, READ), arg_indirect(q_bc, bn, 2, READ)],
                 _k_proxy_bc),
        ]
    handles = {"q": q, "q_old": q_old, "grad": grad, "res": res, "dt_loc": dt_loc,
               "dt_min": dt_mins, "rms": rmss, "x": x, "w": w, "lim": lim, "aux": aux,
               "vol": vol, "q_bc": q_bc}
    return program, handles
