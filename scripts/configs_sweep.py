"""Measure every BASELINE.json config on one B200 (the bench line covers
configs[1]); one JSON line per measurement, for profiles/.

    python scripts/configs_sweep.py [--which 1 3 4 5] [--reps 20]

1  edge flux (indirect INC over edge->node) on ~100K-node meshes: the Kuhn
   3-D grid N=47 (700,534 edges) and the reference generator gen_mesh(316)
   (300,200 edges); per schedule, and the CPU oracle on gen_mesh(316).
3  the 94^3 proxy iteration: random numbering vs CM renumbering, and
   auto-SoA (default) / all-AoS / all-SoA layouts; per-loop ms and GB/s.
4  the ~8M-edge mesh (139^3, 7,998,894 edges) on ONE GPU (the per-GPU
   baseline of the 2/4/8-GPU runs).
5  colouring stress: a 1M-edge random mesh with 8 hub nodes; plan shape
   (blocks, colours, blocks per colour) and edge-flux time per schedule.
"""
import argparse
import json
import statistics
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))

import numpy as np                                  # noqa: E402

import paper_1403_7209_b200 as ml                   # noqa: E402
from paper_1403_7209_b200 import apps               # noqa: E402
from paper_1403_7209_b200.executor import compile_program  # noqa: E402
from paper_1403_7209_b200.plan import plan_stats    # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--which", type=int, nargs="+", default=[1, 3, 4, 5])
ap.add_argument("--reps", type=int, default=20)
args = ap.parse_args()


def loop_times(prog, mesh, cfg, reps):
    cp = compile_program(prog, mesh, cfg)
    for _ in range(3):
        cp.run(False, True)
    per = {e.loop.name: [] for e in cp.entries}
    for _ in range(reps):
        for e, t in zip(cp.entries, cp.run(False, True)):
            per[e.loop.name].append(t)
    return {e.loop.name: {"ms": round(1e3 * statistics.median(per[e.loop.name]), 4),
                          "gbs_alg": round(e.alg / statistics.median(per[e.loop.name]) / 1e9, 1),
                          "b_alg": e.alg}
            for e in cp.entries}, cp


def emit(**kw):
    print(json.dumps(kw), flush=True)


if 1 in args.which:
    for name, gen in (("kuhn47", lambda: apps.gen_kuhn_mesh(47, seed=0)),
                      ("gen_mesh316", lambda: apps.gen_mesh(316))):
        mesh = gen()
        apps.shuffle_mesh(mesh, seed=1)
        prog, h = apps.build_diffusion(mesh, 1, dtype="float64")
        ml.renumber_mesh(mesh)
        for sched in ("gather", "pfold", "colour"):
            t, _ = loop_times(prog, mesh, ml.BackendConfig(device=0, inc_schedule=sched), args.reps)
            e = mesh.sets["edges"].size
            emit(config=1, mesh=name, edges=e, schedule=sched, loops=t,
                 edge_flux_edges_per_s=e / (t["edge_flux"]["ms"] * 1e-3))
    from oracle import serial
    mesh = apps.gen_mesh(316)
    prog, h = apps.build_diffusion(mesh, 1, dtype="float64")
    t0 = time.perf_counter()
    serial.run_loop(prog[1])
    dt = time.perf_counter() - t0
    emit(config=1, mesh="gen_mesh316", cpu_oracle_edge_flux_s=dt,
         cpu_edges_per_s=mesh.sets["edges"].size / dt, cores=1,
         note="oracle/serial.py restating reference run_serial")

if 3 in args.which:
    for renumber in (False, True):
        for soa, label in ((4, "auto-SoA (dim>4)"), (None, "all AoS"), (0, "all SoA")):
            mesh = apps.gen_hex_mesh(94, seed=0, auto_soa_threshold=soa)
            apps.shuffle_mesh(mesh, seed=1)
            prog, h = apps.build_hydra_proxy(mesh, steps=1, seed=0)
            if renumber:
                ml.renumber_mesh(mesh)
            for sched in ("gather", "pfold"):
                t, _ = loop_times(prog, mesh, ml.BackendConfig(device=0, inc_schedule=sched), args.reps)
                emit(config=3, renumbered=renumber, layout=label, schedule=sched, loops=t,
                     iteration_ms=round(sum(v["ms"] for v in t.values()), 4))

if 4 in args.which:
    mesh = apps.gen_hex_mesh(139, seed=0)
    apps.shuffle_mesh(mesh, seed=1)
    prog, h = apps.build_hydra_proxy(mesh, steps=1, seed=0)
    ml.renumber_mesh(mesh)
    for sched in ("gather", "pfold"):
        t, cp = loop_times(prog, mesh, ml.BackendConfig(device=0, inc_schedule=sched), args.reps)
        it = sum(v["ms"] for v in t.values())
        emit(config=4, mesh="hex139", edges=mesh.sets["edges"].size, schedule=sched, loops=t,
             iteration_ms=round(it, 4), edges_per_s=mesh.sets["edges"].size / (it * 1e-3), n_gpus=1)

if 5 in args.which:
    mesh = apps.gen_hub_mesh(250_000, 1_000_000, n_hubs=8, hub_share=0.02, seed=3)
    prog, h = apps.build_diffusion(mesh, 1, dtype="float64")
    loop = prog[1]
    for bs in (256,):
        p = ml.plan_for(loop, mesh, bs)
        st = plan_stats(p)
        bpc = np.diff(p.color_offsets)
        for sched in ("gather", "pfold", "colour"):
            t, _ = loop_times([loop], mesh, ml.BackendConfig(device=0, inc_schedule=sched,
                                                             block_size=bs), args.reps)
            emit(config=5, mesh="hub 250k nodes / 1M edges, 8 hubs", block_size=bs, nb=st.nb,
                 nc=st.nc, blocks_per_colour_min=int(bpc.min()), blocks_per_colour_max=int(bpc.max()),
                 schedule=sched, edge_flux=t["edge_flux"])
