"""Multi-rank owner-compute protocol on CPU: world_size 2 (and 3), gloo.

The host side of the multi-GPU layer — layout, local numbering
[owned | exec | non-exec], iteration prefixes, lazy halo exchange with dirty
bits, rank-ordered reduction folding, final gather — runs for real across
processes; only the per-rank loop execution is the CPU oracle (injected),
since this container has no GPU.  Results must equal the reference serial
golden vectors bit for bit (int64) — the reference's own multi-rank
equivalence contract (tests/test_executor.py:137-186).
"""
from __future__ import annotations

import os
import socket
import sys
from pathlib import Path

import numpy as np
import pytest

ROOT = Path(__file__).resolve().parent.parent


def _free_port() -> int:
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


class OracleRank:
    """Executes a RankProgram's local loops with the CPU oracle (test-only)."""

    def __init__(self, rp, config):
        self.rp = rp

    def run_loop(self, i: int) -> float:
        from oracle import serial
        rp = self.rp
        loop = rp.loops[i]
        rp.reset_partials(i)
        s = loop.iter_set.name
        n_own, n_exec = rp.n_owned[s], rp.n_exec[s]
        acc = serial.element_views(loop)
        for e in range(n_own):
            loop.kernel(*[a(e) for a in acc])
        red = [j for j, a in enumerate(loop.args) if a.kind == "global" and a.mode.name != "READ"]
        acc2 = list(acc)
        for j in red:
            g = loop.args[j].glob
            scratch = serial.reduce_identity(loop.args[j].mode.name, g.dtype, g.dim)
            acc2[j] = lambda e, s=scratch: s
        for e in range(n_own, n_exec):
            loop.kernel(*[a(e) for a in acc2])
        return 0.0

    def pack(self, name, ids):
        return self.rp.dats[name].fetch()[ids]

    def unpack(self, name, ids, rows):
        d = self.rp.dats[name]
        vals = d.fetch()
        vals[ids] = rows
        d.put(vals)


def _worker(rank, world, port, case, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK=str(rank),
                      WORLD_SIZE=str(world))
    sys.path[:0] = [str(ROOT), str(ROOT / "tests")]
    import torch.distributed as dist
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import _cases
        import paper_1403_7209_b200 as ml
        from paper_1403_7209_b200.multigpu import run_program_distributed
        app, n, dtype, steps, part = case
        if app == "fuzz":
            mesh, loop = _cases.random_loop_mesh(np.random.default_rng(n), max_elems=300)
            prog, res = [loop], None
        elif app == "reads":
            mesh = ml.Mesh()
            from paper_1403_7209_b200 import apps
            mesh = apps.gen_mesh(4)
            prog = _read_program(mesh, steps)
        elif app == "proxy":
            from paper_1403_7209_b200 import apps
            mesh = apps.gen_hex_mesh(n, seed=7)
            prog, h = apps.build_hydra_proxy(mesh, steps=steps, seed=7)
        elif app == "repeat":
            mesh, prog, h = _cases.build_app("diffusion", n, dtype, 1)
        else:
            mesh, prog, h = _cases.build_app(app, n, dtype, steps)
        cfg = ml.BackendConfig(nranks=world, partitioner=part)
        if app == "repeat":
            # one run_program call per time step: the cached rank setup is reused
            # and a host write to a global dat between calls is seen
            from paper_1403_7209_b200 import multigpu
            setups = []
            for k in range(steps):
                result = run_program_distributed(prog, mesh, cfg, executor_factory=OracleRank)
                setups.append(id(next(iter(mesh.__dict__["_ml_dist"].values()))[1][0]))
                u = mesh.dats["u"].fetch()
                u[::5] += k + 1
                mesh.dats["u"].put(u)
            out = {"u": mesh.dats["u"].fetch(), "res": np.array([g.value for g in h["residuals"]]),
                   "setups": len(set(setups))}
            q.put((rank, out, result.messages))
            return
        result = run_program_distributed(prog, mesh, cfg, executor_factory=OracleRank)
        if app == "proxy":
            out = {"q": h["q"].fetch(), "rms": np.array([r.value for r in h["rms"]]),
                   "loops": [r.loop for r in result.perf]}
        elif app == "fuzz":
            out = {"vals": mesh.dats["vals"].fetch()}
        elif app == "reads":
            out = {}
        else:
            out = _cases.app_results(app, h)
        q.put((rank, out, result.messages))
    except Exception as err:          # surface worker failures to the parent
        import traceback
        q.put((rank, traceback.format_exc(), -1))
    finally:
        dist.destroy_process_group()


def _read_program(mesh, repeats):
    import paper_1403_7209_b200 as ml
    from paper_1403_7209_b200.kernels import device_kernel
    nodes, edges = mesh.sets["nodes"], mesh.sets["edges"]
    en = mesh.maps["edge_nodes"]
    u = mesh.decl_dat("u", nodes, 1, "float64", np.zeros(nodes.size))
    acc = mesh.decl_dat("acc", edges, 1, "float64", np.zeros(edges.size))

    @device_kernel("set_one")
    def init(v):
        v[0] = 1.0

    @device_kernel("gather_pair")
    def gather(a, b, out):
        out[0] = out[0] + a[0] + b[0]
    w = ml.Loop("init", nodes, [ml.arg_direct(u, ml.WRITE)], init)
    r = ml.Loop("gather", edges, [ml.arg_indirect(u, en, 1, ml.READ), ml.arg_indirect(u, en, 2, ml.READ),
                                  ml.arg_direct(acc, ml.INC)], gather)
    return [w] + [r] * repeats


def _run(case, world=2):
    import multiprocessing as mp
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, case, q)) for r in range(world)]
    for p in procs:
        p.start()
    outs = [q.get(timeout=240) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
    for rank, out, msgs in outs:
        if msgs < 0:
            raise AssertionError(f"rank {rank} failed:\n{out}")
    return sorted(outs, key=lambda x: x[0])


@pytest.mark.parametrize("case", [
    ("diffusion", 8, "int64", 3, "trivial"),
    ("diffusion", 8, "int64", 3, "rcb"),
    ("cell-area", 6, "int64", 0, "rcb"),
])
def test_two_ranks_match_reference_serial_bit_exact(case):
    from conftest import golden
    g = golden("exec.npz")
    app, n, dtype, steps, _ = case
    name = f"{app}_n{n}_{dtype}_s{steps}"
    outs = _run(case)
    for rank, out, msgs in outs:
        assert (msgs > 0) == (app == "diffusion")   # cell-area never reads a dirty halo
        for k, v in out.items():
            np.testing.assert_array_equal(v, g[f"exec/{name}/{k}"], f"rank {rank} {k}")


def test_three_ranks_fuzz_mesh():
    from conftest import golden
    g = golden("exec.npz")
    case = next(c for c in g.index if c["name"] == "fuzz0")
    outs = _run(("fuzz", case["seed"], "int64", 0, "trivial"), world=3)
    for rank, out, _ in outs:
        np.testing.assert_array_equal(out["vals"], g["exec/fuzz0/vals"])


def test_consecutive_reads_move_no_extra_messages():
    """reference tests/test_executor.py:217-239: re-reads of clean data exchange nothing."""
    m1 = _run(("reads", 0, "float64", 1, "trivial"))[0][2]
    m3 = _run(("reads", 0, "float64", 3, "trivial"))[0][2]
    assert m1 > 0 and m1 == m3


def test_two_ranks_chained_proxy_matches_serial():
    """The proxy's iflux+vflux chain runs as one loop per rank (its halo is the
    union of both loops'); q and rms within the reference rtol of the serial
    oracle running the unchained program on one process."""
    import paper_1403_7209_b200 as ml  # noqa: F401
    from oracle import serial
    from paper_1403_7209_b200 import apps
    mesh = apps.gen_hex_mesh(5, seed=7)
    prog, h = apps.build_hydra_proxy(mesh, steps=2, seed=7)
    serial.run_program(prog)
    for rank, out, msgs in _run(("proxy", 5, "float64", 2, "rcb")):
        assert msgs > 0 and "iflux+vflux" in out["loops"] and "vflux" not in out["loops"]
        ref = h["q"].fetch()
        np.testing.assert_allclose(out["q"], ref, rtol=1e-12, atol=1e-12 * np.abs(ref).max())
        np.testing.assert_allclose(out["rms"], [r.value for r in h["rms"]], rtol=1e-12)


def test_repeated_run_program_reuses_rank_setup_and_sees_host_writes():
    """a multi-rank program run once per time step must not rebuild
    its layout / rank program / IPC mappings, and must start every run from
    the global mesh's current values."""
    import _cases
    from oracle import serial
    mesh, prog, h = _cases.build_app("diffusion", 8, "int64", 1)
    for k in range(3):
        serial.run_program(prog)
        u = mesh.dats["u"].fetch()
        u[::5] += k + 1
        mesh.dats["u"].put(u)
    outs = _run(("repeat", 8, "int64", 3, "rcb"))
    for _rank, out, _msgs in outs:
        assert out["setups"] == 1
        np.testing.assert_array_equal(out["u"], mesh.dats["u"].fetch())
        np.testing.assert_array_equal(out["res"], [g.value for g in h["residuals"]])
