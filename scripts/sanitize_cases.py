"""Small programs covering every kernel family, for compute-sanitizer
(memcheck / racecheck / synccheck / initcheck; scripts/sanitize.sh).

Each case runs through the public API on tiny meshes: the diffusion app
(int64) and the Hydra proxy (float64) under every INC schedule, a hub mesh
(split hub rows: k_gather_hubs, k_fold_parts), the colour schedule with the
per-phase callback, streamed host residency, CUDA-graph replay and an empty
iteration set.  ``--ranks`` adds the owner-compute path with 2 ranks sharing
the GPU (NVLink IPC halo puts, delivery/credit flags, NVLink reductions).
"""
from __future__ import annotations

import argparse
import os
import sys
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))

import paper_1403_7209_b200 as ml          # noqa: E402
from paper_1403_7209_b200 import apps       # noqa: E402


def single_gpu():
    for sched in ("auto", "gather", "pfold", "colour"):
        mesh = apps.gen_mesh(10)
        prog, h = apps.build_diffusion(mesh, 2, dtype="int64")
        ml.run_program(prog, mesh, ml.BackendConfig(inc_schedule=sched, block_size=32))
        mesh = apps.gen_hex_mesh(6, seed=1)
        apps.shuffle_mesh(mesh, seed=2)
        prog, h = apps.build_hydra_proxy(mesh, steps=1, seed=1)
        ml.renumber_mesh(mesh)
        ml.run_program(prog, mesh, ml.BackendConfig(inc_schedule=sched))
        print("ok", sched, flush=True)
    mesh = apps.gen_hex_mesh(5, seed=3)
    prog, h = apps.build_hydra_proxy(mesh, steps=1, seed=3)
    for kw in ({"use_graph": True}, {"residency": "host", "use_graph": True}, {"residency": "host"},
               {"chain_loops": False}, {"phase_callback": lambda name, c: None, "inc_schedule": "colour"}):
        ml.run_program(prog, mesh, ml.BackendConfig(**kw))
        print("ok", sorted(kw), flush=True)
    for sched in ("gather", "pfold"):                       # hub rows (> 128 incidences)
        mesh = apps.gen_hub_mesh(2000, 20000, n_hubs=4, hub_share=0.1, seed=4)
        m = mesh.maps["edge_nodes"]
        acc = mesh.decl_dat("acc", m.to_set, 1, "int64", np.zeros(m.to_set.size, np.int64))
        from paper_1403_7209_b200.kernels import device_kernel

        @device_kernel("inc_one_2")
        def inc(a, b):
            a[0] += 1
            b[0] += 1
        loop = ml.Loop("hub", m.from_set, [ml.arg_indirect(acc, m, 1, ml.INC),
                                           ml.arg_indirect(acc, m, 2, ml.INC)], inc)
        ml.run_program([loop], mesh, ml.BackendConfig(inc_schedule=sched))
        print("ok hubs", sched, flush=True)
    mesh = ml.Mesh()
    nodes = mesh.decl_set("nodes", 4)
    none = mesh.decl_set("none", 0)
    z = mesh.decl_dat("z", none, 1, "int64", [])
    total = ml.Global(np.int64(1))
    ml.run_program([ml.Loop("cnt", none, [ml.arg_direct(z, ml.READ), ml.arg_global(total, ml.INC)],
                            apps._k_sum)], mesh, ml.BackendConfig())
    print("ok empty", flush=True)


def ranks(world: int = 2):
    """Owner-compute run with `world` ranks sharing GPU 0 (spawned processes)."""
    import multiprocessing as mp
    import socket
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    ctx = mp.get_context("spawn")
    procs = [ctx.Process(target=_rank_main, args=(r, world, port)) for r in range(world)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(600)
    codes = [p.exitcode for p in procs]
    if any(codes):
        raise SystemExit(f"rank exit codes {codes}")
    print("ok ranks", world, flush=True)


def _rank_main(rank, world, port):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK=str(rank),
                      WORLD_SIZE=str(world), LOCAL_RANK="0", ML_DEVICE="0", ML_TRANSPORT="gloo")
    mesh = apps.gen_hex_mesh(8, seed=5)
    prog, h = apps.build_hydra_proxy(mesh, steps=2, seed=5)
    ml.renumber_mesh(mesh)
    ml.run_program(prog, mesh, ml.BackendConfig(device=0, nranks=world, partitioner="rcb"))
    import torch.distributed as dist
    dist.barrier()
    dist.destroy_process_group()


if __name__ == "__main__":
    ap = argparse.ArgumentParser()
    ap.add_argument("--ranks", type=int, default=0)
    args = ap.parse_args()
    if args.ranks:
        ranks(args.ranks)
    else:
        single_gpu()
