"""Multi-rank owner-compute execution ON THE GPU: 2 and 3 processes sharing one
B200 (the gpurun box has one GPU; NCCL refuses two ranks on one device, so the
halo rows travel host-staged over gloo — everything else is the production
path: local meshes, ml_pack_rows/ml_unpack_rows, coloured kernels with
iteration prefixes and reduction limits).  Results must equal the reference
serial golden vectors bit for bit (int64) and the oracle within 1e-12 (f64)."""
from __future__ import annotations

import os
import socket
import sys
from pathlib import Path

import numpy as np
import pytest

pytestmark = pytest.mark.gpu
ROOT = Path(__file__).resolve().parent.parent


def _free_port() -> int:
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _worker(rank, world, port, case, q, executor="stream"):
    halo = "p2p"
    if executor.endswith("+copy"):
        executor, halo = executor[:-5], "copy"
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK=str(rank),
                      WORLD_SIZE=str(world), LOCAL_RANK="0", ML_TRANSPORT="gloo",
                      ML_RANK_EXECUTOR=executor, ML_HALO=halo)
    sys.path[:0] = [str(ROOT), str(ROOT / "tests")]
    import torch.distributed as dist
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import _cases
        import paper_1403_7209_b200 as ml
        from paper_1403_7209_b200 import apps
        app, n, dtype, steps, part, sched = case
        if app == "proxy":
            mesh = apps.gen_hex_mesh(n, seed=5)
            prog, h = apps.build_hydra_proxy(mesh, steps=steps, seed=5)
            ml.renumber_mesh(mesh)
        else:
            mesh, prog, h = _cases.build_app(app, n, dtype, steps)
        cfg = ml.BackendConfig(nranks=world, partitioner=part, device=0, inc_schedule=sched)
        result = ml.run_program(prog, mesh, cfg)
        if app == "proxy":
            import paper_1403_7209_b200.multigpu as mg
            out = {"q": h["q"].fetch(), "rms": np.array([g.value for g in h["rms"]]),
                   "dt": np.array([g.value for g in h["dt_min"]]), "overlapped": list(mg._LAST_OVERLAPPED)}
        else:
            out = _cases.app_results(app, h)
        need_nvlink = executor == "stream" and halo == "p2p" and world > 1
        q.put((rank, out, result.messages if not need_nvlink or _nvlink_used() else -2))
    except Exception:
        import traceback
        q.put((rank, traceback.format_exc(), -1))
    finally:
        dist.destroy_process_group()


def _nvlink_used() -> bool:
    import paper_1403_7209_b200.multigpu as mg
    return bool(getattr(mg, "_LAST_HALO_PATH", "") == "nvlink")


def _run(case, world=2, executor="stream"):
    import multiprocessing as mp
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, case, q, executor))
             for r in range(world)]
    for p in procs:
        p.start()
    outs = [q.get(timeout=600) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
    for rank, out, msgs in outs:
        if msgs == -2:
            raise AssertionError(f"rank {rank}: the NVLink (IPC) halo path was not used")
        if msgs < 0:
            raise AssertionError(f"rank {rank} failed:\n{out}")
    return sorted(outs, key=lambda x: x[0])


@pytest.mark.parametrize("world,part,sched,executor", [
    (2, "rcb", "gather", "stream"), (3, "trivial", "gather", "stream"), (2, "rcb", "colour", "stream"),
    (2, "rcb", "gather", "stream+copy"), (3, "trivial", "pfold", "stream+copy"),
    (3, "trivial", "colour", "host"), (2, "trivial", "colour", "host"),
    (2, "rcb", "pfold", "stream")])
def test_ranks_on_device_match_reference_int64(world, part, sched, executor):
    from conftest import golden
    g = golden("exec.npz")
    outs = _run(("diffusion", 8, "int64", 3, part, sched), world, executor)
    for rank, out, msgs in outs:
        assert msgs > 0
        for k, v in out.items():
            np.testing.assert_array_equal(v, g[f"exec/diffusion_n8_int64_s3/{k}"], f"rank {rank} {k}")


@pytest.mark.parametrize("sched,executor", [("gather", "stream"), ("gather", "stream+copy"),
                                            ("colour", "host"), ("pfold", "stream"), ("auto", "stream+copy")])
def test_proxy_two_ranks_on_device_vs_oracle(sched, executor):
    import paper_1403_7209_b200 as ml
    from oracle import bulk
    from paper_1403_7209_b200 import apps
    mesh = apps.gen_hex_mesh(12, seed=5)
    prog, h = apps.build_hydra_proxy(mesh, steps=2, seed=5)
    ml.renumber_mesh(mesh)
    bulk.run_program(prog)
    outs = _run(("proxy", 12, "float64", 2, "rcb", sched), 2, executor)
    ref_q = h["q"].fetch()
    for rank, out, _ in outs:
        if executor.startswith("stream") and sched in ("pfold", "auto"):
            # the fused flux loop runs as pfold, its pass-1 rows split around the exchange
            assert ("iflux+vflux", "pfold") in out["overlapped"], out["overlapped"]
        np.testing.assert_allclose(out["q"], ref_q, rtol=1e-12, atol=1e-12 * np.abs(ref_q).max())
        np.testing.assert_allclose(out["rms"], [r.value for r in h["rms"]], rtol=1e-12)
        np.testing.assert_array_equal(out["dt"], [r.value for r in h["dt_min"]])


def _graph_worker(port, q):
    """One NCCL rank: a CUDA-graph-captured rank step (loops, NCCL all-gather of
    the reductions, rank fold) replayed twice must equal two eager steps."""
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK="0", WORLD_SIZE="1",
                      LOCAL_RANK="0")
    sys.path[:0] = [str(ROOT), str(ROOT / "tests")]
    try:
        import paper_1403_7209_b200 as ml
        from paper_1403_7209_b200 import apps
        from paper_1403_7209_b200.multigpu import setup_distributed
        outs = []
        for graphed in (False, True):
            mesh = apps.gen_hex_mesh(14, seed=6)
            prog, h = apps.build_hydra_proxy(mesh, steps=1, seed=6)
            ml.renumber_mesh(mesh)
            cfg = ml.BackendConfig(nranks=1, partitioner="rcb", device=0)
            rp, dev, tr, layout, cfg = setup_distributed(prog, mesh, cfg)
            assert tr.name == "nccl"
            dev.run()
            dev.finish()
            if graphed:
                dev.capture()
                dev.replay()
                dev.replay()
            else:
                dev.run()
                dev.run()
            dev.finish()
            outs.append((rp.dats["q"].fetch(), [v.buffer.copy() for v in rp.values.values()]))
        q.put((outs[0][0], outs[1][0], outs[0][1], outs[1][1], None))
    except Exception:
        import traceback
        q.put((None, None, None, None, traceback.format_exc()))


def test_rank_step_cuda_graph_with_nccl_matches_eager():
    import multiprocessing as mp
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    p = ctx.Process(target=_graph_worker, args=(_free_port(), q))
    p.start()
    a, b, va, vb, err = q.get(timeout=600)
    p.join(timeout=60)
    assert err is None, err
    np.testing.assert_array_equal(a, b)
    for x, y in zip(va, vb):
        np.testing.assert_array_equal(x, y)


def _timeout_worker(rank, port, q):
    """Rank 0 runs a program whose second loop needs rank 1's halo rows; rank 1
    never runs it: the NVLink wait must expire and surface as ExchangeTimeout
    (reference executor.py:343-359), not hang."""
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK=str(rank), WORLD_SIZE="2",
                      LOCAL_RANK="0", ML_TRANSPORT="gloo", ML_HALO="p2p")
    sys.path[:0] = [str(ROOT), str(ROOT / "tests")]
    import torch.distributed as dist
    dist.init_process_group("gloo", rank=rank, world_size=2)
    try:
        import paper_1403_7209_b200 as ml
        from paper_1403_7209_b200 import apps
        from paper_1403_7209_b200.apps import _k_copy, _k_edge_flux
        from paper_1403_7209_b200.executor import ExchangeTimeout
        from paper_1403_7209_b200.multigpu import setup_distributed
        mesh = apps.gen_mesh(10)
        nodes, edges = mesh.sets["nodes"], mesh.sets["edges"]
        en = mesh.maps["edge_nodes"]
        u = mesh.decl_dat("u", nodes, 1, "float64", np.arange(nodes.size, dtype=float))
        u0 = mesh.decl_dat("u0", nodes, 1, "float64", np.ones(nodes.size))
        fl = mesh.decl_dat("fl", nodes, 1, "float64", np.zeros(nodes.size))
        prog = [ml.Loop("write_u", nodes, [ml.arg_direct(u0, ml.READ), ml.arg_direct(u, ml.WRITE)], _k_copy),
                ml.Loop("flux", edges, [ml.arg_indirect(u, en, 1, ml.READ), ml.arg_indirect(u, en, 2, ml.READ),
                                        ml.arg_indirect(fl, en, 1, ml.INC), ml.arg_indirect(fl, en, 2, ml.INC)],
                        _k_edge_flux)]
        cfg = ml.BackendConfig(nranks=2, partitioner="trivial", device=0, timeout_ms=300.0)
        rp, dev, tr, layout, cfg = setup_distributed(prog, mesh, cfg)
        assert dev.nvlink is not None
        if rank == 0:
            dev.run()
            dev.run()                          # the second run exchanges u (dirty after run 1)
            try:
                dev.finish()
                q.put((rank, "no timeout raised"))
            except ExchangeTimeout as ex:
                q.put((rank, "ok" if "no message from rank 1" in str(ex) and "'u'" in str(ex) else str(ex)))
        else:
            q.put((rank, "ok"))
    except Exception:
        import traceback
        q.put((rank, traceback.format_exc()))


def test_nvlink_halo_wait_times_out_as_exchange_timeout():
    import multiprocessing as mp
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_timeout_worker, args=(r, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    outs = dict(q.get(timeout=300) for _ in range(2))
    for p in procs:
        p.join(timeout=30)
        if p.is_alive():
            p.kill()
    assert outs == {0: "ok", 1: "ok"}, outs


def _graph2_worker(rank, port, q):
    """Two ranks on one GPU, NVLink (IPC) halos and reductions: a captured rank
    step replayed twice equals two eager steps, on both ranks."""
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK=str(rank), WORLD_SIZE="2",
                      LOCAL_RANK="0", ML_TRANSPORT="gloo", ML_HALO="p2p")
    sys.path[:0] = [str(ROOT), str(ROOT / "tests")]
    import torch.distributed as dist
    dist.init_process_group("gloo", rank=rank, world_size=2)
    try:
        import paper_1403_7209_b200 as ml
        from paper_1403_7209_b200 import apps
        from paper_1403_7209_b200.multigpu import setup_distributed
        outs = []
        for graphed in (False, True):
            mesh = apps.gen_hex_mesh(12, seed=6)
            prog, h = apps.build_hydra_proxy(mesh, steps=1, seed=6)
            ml.renumber_mesh(mesh)
            cfg = ml.BackendConfig(nranks=2, partitioner="rcb", device=0)
            rp, dev, tr, layout, cfg = setup_distributed(prog, mesh, cfg)
            assert dev.nvlink is not None and dev.nvreduce is not None
            dev.run()
            dev.finish()
            if graphed:
                dev.capture()
                dev.replay()
                dev.replay()
            else:
                dev.run()
                dev.run()
            dev.finish()
            outs.append((rp.dats["q"].fetch()[: rp.n_owned["nodes"]],
                         [v.buffer.copy() for v in rp.values.values()]))
        same = (np.array_equal(outs[0][0], outs[1][0])
                and all(np.array_equal(a, b) for a, b in zip(outs[0][1], outs[1][1])))
        q.put((rank, "ok" if same else "graph replay differs from eager steps"))
    except Exception:
        import traceback
        traceback.print_exc()
        q.put((rank, traceback.format_exc()[-3000:]))


def test_two_rank_graph_with_nvlink_paths_matches_eager():
    import multiprocessing as mp
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_graph2_worker, args=(r, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    outs = dict(q.get(timeout=600) for _ in range(2))
    for p in procs:
        p.join(timeout=60)
    assert outs == {0: "ok", 1: "ok"}, outs
