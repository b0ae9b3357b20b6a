"""Benchmark: one Hydra-shaped solver iteration per step on B200 (BASELINE.json configs[1]).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
                    [--workload proxy|diffusion] [--grid 94] [--inc-schedule tuned|gather|pfold|...]

Workload (default): ``build_hydra_proxy`` on the Rotor37-sized 3-D grid
(94^3 = 830,584 nodes, 2,465,244 edges), numbered randomly (an unstructured
mesh as read from disk) and then Cuthill–McKee renumbered; float64, one
iteration = save -> dt_calc (MIN) -> grad_edge -> iflux -> vflux -> update
(SUM) -> bc (7 op_par_loops; iflux and vflux run chained as one fused loop
``iflux+vflux``, chain.py).  Inputs (~570 MB of dats + maps) exceed the
126 MB L2, so no flush is needed between steps.

Metric (BASELINE.json): edges/s (whole job) and time per solver iteration,
plus achieved HBM GB/s vs the measured peak for the dominant loop (the one
containing vflux).

* ``value``      edges/s with all state resident in HBM: K back-to-back CUDA
                 graph replays of the iteration, CUDA events on the library
                 stream (N=1); max over ranks (N>1).
* ``e2e``        the same metric through the public API with HOST buffers:
                 every step ``run_program(..., residency="host")`` uploads
                 every input dat of the iteration from pinned host memory and
                 downloads every dat it writes plus the reductions; uploads,
                 loops and downloads overlap on three streams.  ``e2e.pcie``:
                 measured pinned H2D / D2H bandwidth and the step times they
                 bound (all inputs through H2D; + the serial D2H).
* ``roofline``   vflux (``iflux+vflux`` chained): B_alg / its mean device time in
                 the steady-state CUDA graph (a sequential capture of the same
                 program with a timing event between loops, K replays); the
                 per-loop ``loops`` table is measured the same way (``eager_ms``:
                 eager launches with events, for comparison).
* ``cpu_baseline`` the stock reference (``meshloop.run_program`` from
                 baseline/_ref) on this host's CPUs in its three modes:
                 serial on the full workload (once), threads (all CPUs) and
                 ranks (power-of-two ranks, RCB) on a ``--cpu-grid`` sample;
                 ``lscpu`` model; value = best per-edge rate.

``--impl reference`` times the stock reference alone (threads backend, all
host CPUs) on the ``--cpu-grid`` sample, one iteration per step, and labels
the workload it ran (rank 0; other ranks exit).
Multi-GPU (torchrun, N>1): RCB owner-compute partition of the same mesh
(strong scaling), one GPU per rank, halos over NVLink peer memory (NCCL
fallback); value = total edges/s.
"""
from __future__ import annotations

import argparse
import ctypes as C
import json
import os
import statistics
import sys
import time
from pathlib import Path

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

from paper_1403_7209_b200.bench_support import (build_workload, clock_sampler, cpu_model,  # noqa: E402
                                                  load_reference, peaks_gbs, reference_modes,
                                                  time_reference, workload_name)

METRIC = "edges/sec and time per solver iteration; achieved HBM GB/s vs peak, 1/2/4/8 B200"


def _port_baseline(args) -> dict:
    """Fallback when the stock reference is not importable: the oracle's
    restatement of reference run_serial (oracle/serial.py) on the sample grid."""
    from oracle import serial
    a = argparse.Namespace(**{**vars(args), "grid": args.cpu_grid})
    mesh, prog, _h, name, _setup = build_workload(a)
    t0 = time.perf_counter()
    serial.run_program(prog)
    dt = time.perf_counter() - t0
    edges = mesh.sets["edges"].size
    return {"value": edges / dt, "unit": "edges/s", "cores": 1, "kind": "port",
            "sample": f"{name} ({edges} edges), one iteration; oracle/serial.py restating reference "
                      f"run_serial (executor.py:206-217) — the stock reference was not importable",
            "sec_per_iteration": dt, "host_cpus": os.cpu_count(), "cpu_model": cpu_model()}


def cpu_baseline(args) -> dict:
    """The stock reference (baseline/_ref ``meshloop.run_program``) on this host's
    CPU, in its three modes: serial on the full bench workload
    (once; ``--cpu-sample-only`` moves it to the sample), threads (nthreads =
    all host CPUs) and ranks (largest power of two <= CPUs, RCB) on the
    ``--cpu-grid`` sample.  ``value`` = the best per-edge rate of the three."""
    R = load_reference()
    if R is None:
        return _port_baseline(args)
    cores = os.cpu_count() or 1
    modes = {}
    sample = argparse.Namespace(**{**vars(args), "grid": args.cpu_grid})
    full = sample if args.cpu_sample_only else args
    for mode, a, warm in (("serial", full, 0), ("threads", sample, 1), ("ranks", sample, 0)):
        mesh, prog, _h, name, _setup = build_workload(a)
        edges = mesh.sets["edges"].size
        sec, calls = time_reference(R, mesh, prog, mode, cores, runs=1, warm=warm)
        cfg = reference_modes(cores)[mode]
        modes[mode] = {"workload": name, "edges": edges, "sec_per_iteration": round(sec, 3),
                       "edges_per_s": edges / sec,
                       "cores": cfg.get("nthreads", cfg.get("nranks", 1)),
                       "config": {"backend": "serial", **cfg},
                       "run_program_calls": calls}
    best = max(modes, key=lambda m: modes[m]["edges_per_s"])
    return {"value": modes[best]["edges_per_s"], "unit": "edges/s", "cores": modes[best]["cores"],
            "kind": "reference", "mode": best,
            "sample": (f"stock meshloop.run_program (baseline/_ref): serial on {modes['serial']['workload']}, "
                       f"threads/ranks on {modes['threads']['workload']}; one iteration each "
                       f"(threads after one untimed plan-building call; ranks includes the "
                       f"reference's per-call layout build and runs the iteration as "
                       f"{modes['ranks']['run_program_calls']} calls so dt_min is folded before "
                       f"update reads it); value = best per-edge rate ({best})"),
            "modes": modes, "host_cpus": cores, "cpu_model": cpu_model()}


def run_reference(args) -> None:
    """``--impl reference``: the stock reference (``meshloop.run_program``,
    threads backend with every host CPU) on a bounded sample of the bench
    workload, one iteration per step; rank 0 only."""
    if int(os.environ.get("RANK", "0")) != 0:
        return
    R = load_reference()
    cores = os.cpu_count() or 1
    sample = argparse.Namespace(**{**vars(args), "grid": args.cpu_grid})
    mesh, prog, _h, name, _setup = build_workload(sample)
    edges = mesh.sets["edges"].size
    secs = []
    if R is not None:
        from paper_1403_7209_b200.foreign import export_mesh, export_program
        ref = export_mesh(mesh, R)
        rprog = export_program(prog, ref, R)
        cfg = R.BackendConfig(**reference_modes(cores)["threads"])
        for k in range(args.warmup + args.steps):
            t0 = time.perf_counter()
            R.run_program(rprog, ref, cfg)
            if k >= args.warmup:
                secs.append(time.perf_counter() - t0)
        kind, par = "reference", f"stock meshloop.run_program, threads backend, nthreads={cores}"
        what = "stock reference meshloop (baseline/_ref)"
    else:
        from oracle import serial
        for k in range(args.warmup + args.steps):
            t0 = time.perf_counter()
            serial.run_program(prog)
            if k >= args.warmup:
                secs.append(time.perf_counter() - t0)
        kind, par, cores = "port", "oracle/serial.py (reference run_serial restated), 1 core", 1
        what = "oracle port (stock reference not importable)"
    sec = statistics.mean(secs)
    value = edges / sec
    cb = {"value": value, "unit": "edges/s", "cores": cores, "kind": kind,
          "sample": f"{name} ({edges} edges), one iteration per step: a bounded sample of the "
                    f"bench workload ({workload_name(args)}) sized for minutes of CPU time; {what}",
          "host_cpus": os.cpu_count(), "cpu_model": cpu_model()}
    line = {"impl": "reference", "metric": METRIC, "value": value, "unit": "edges/s",
            "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": 1e3 * sec, "higher_is_better": True,
            "scaling": "strong", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": {"workload": name, "edges": edges, "parallelism": par,
                       "sample_of": workload_name(args)},
            "cpu_baseline": cb,
            "e2e": {"value": value, "unit": "edges/s", "h2d_bytes_per_step": 0,
                    "d2h_bytes_per_step": 0}}
    print(json.dumps(line))


def _replay_seconds(cp) -> float:
    t0 = time.perf_counter()
    cp.replay(1)
    return time.perf_counter() - t0


def pcie_bounds(h2d: int, d2h: int) -> dict:
    """Pinned host<->device copy bandwidth on this box (256 MB each way, CUDA
    events, best of 3) and the e2e step time it bounds: inputs cannot all be
    on the device before the H2D stream has moved them, so an e2e step takes
    at least h2d / H2D bandwidth (the D2H of early-written dats overlaps it)."""
    import torch
    n = 256 << 20
    host = torch.empty(n, dtype=torch.uint8).pin_memory()
    dev = torch.empty(n, dtype=torch.uint8, device="cuda")
    out = {}
    for name, dst, src in (("h2d_gbs", dev, host), ("d2h_gbs", host, dev)):
        dst.copy_(src, non_blocking=True)          # untimed: first-touch / mapping costs
        torch.cuda.synchronize()
        best = 0.0
        for _ in range(3):
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record()
            dst.copy_(src, non_blocking=True)
            b.record()
            b.synchronize()
            best = max(best, n / (a.elapsed_time(b) * 1e-3) / 1e9)
        out[name] = round(best, 1)
    out["h2d_bound_ms"] = round(h2d / (out["h2d_gbs"] * 1e9) * 1e3, 3)
    out["serial_bound_ms"] = round((h2d / out["h2d_gbs"] + d2h / out["d2h_gbs"]) / 1e6, 3)
    return out


def scaling_base(args) -> dict:
    """The N=1 point of the multi-GPU curve: ``--scale-grid`` (default 139^3,
    BASELINE configs[3]) through the same rank executor the 2/4/8-GPU runs use
    (StreamRank, world size 1, RCB layout of one rank, CUDA-graph rank step),
    device time only.  ``value`` of this line stays the configs[1] number."""
    from paper_1403_7209_b200.multigpu import bench_distributed
    env = {"RANK": "0", "LOCAL_RANK": "0", "WORLD_SIZE": "1", "MASTER_ADDR": "127.0.0.1",
           "MASTER_PORT": str(_free_port())}
    saved = {k: os.environ.get(k) for k in env}
    os.environ.update(env)
    try:
        a = argparse.Namespace(**{**vars(args), "grid": args.scale_grid, "inc_schedule": "auto"})
        line = bench_distributed(a, METRIC, emit=False, with_e2e=False)
    finally:
        for k, v in saved.items():
            if v is None:
                os.environ.pop(k, None)
            else:
                os.environ[k] = v
    return {"workload": line["config"]["workload"], "edges": line["config"]["edges"],
            "value": line["value"], "unit": "edges/s", "ms_per_step": line["ms_per_step"],
            "n_gpus": 1, "executor": "StreamRank (multigpu.py), world size 1",
            "cuda_graph": line["config"]["cuda_graph"],
            "roofline_frac": line["roofline"]["frac"], "loops_ms": line["loops_ms_rank0"]}


def run_ours(args) -> None:
    world = int(os.environ.get("WORLD_SIZE", "1"))
    if world > 1 or args.gpus > 1:
        from paper_1403_7209_b200.multigpu import bench_distributed
        bench_distributed(args, METRIC)
        return
    import paper_1403_7209_b200 as ml
    from paper_1403_7209_b200 import _native as N
    from paper_1403_7209_b200.device import pin_mesh
    from paper_1403_7209_b200.executor import compile_program

    mesh, prog, h, wname, setup = build_workload(args)
    edges = mesh.sets["edges"].size
    table = None
    sched = args.inc_schedule
    if args.schedule_table:
        table = dict(kv.split("=", 1) for kv in args.schedule_table.split(","))
        sched = "gather" if sched == "tuned" else sched
    elif sched == "tuned":
        # per-loop INC schedule chosen on the device before timing (OP2-style
        # auto-tuning, tuner.tune_schedule): gather vs primary fold
        from paper_1403_7209_b200.tuner import tune_schedule
        t0 = time.perf_counter()
        res = tune_schedule(prog, mesh, ("gather", "pfold"), ml.BackendConfig(device=0), repeats=3)
        table = dict(res.best)
        setup["tune_s"] = round(time.perf_counter() - t0, 3)
        sched = "gather"
    cfg = ml.BackendConfig(device=0, use_graph=True, inc_schedule=sched, inc_schedule_table=table)
    t0 = time.perf_counter()
    cp = compile_program(prog, mesh, cfg)
    setup["plans_and_upload_s"] = round(time.perf_counter() - t0, 3)
    info = N.device_info()

    # -- device-resident throughput: K graph replays, CUDA events ----------------------
    cp.replay(args.warmup)
    timer = C.c_void_p()
    N.check(N.lib().ml_timer_create(C.byref(timer)))
    ms = C.c_float()
    with clock_sampler(0) as clk:
        # nvidia-smi needs ~0.2 s to start: keep the GPU busy (untimed) until it samples
        time.sleep(0.3)
        cp.replay(max(20, int(0.3 / max(_replay_seconds(cp), 1e-4))))
        N.check(N.lib().ml_synchronize())
        N.check(N.lib().ml_timer_start(timer))
        cp.replay(args.steps)
        N.check(N.lib().ml_timer_stop(timer, C.byref(ms)))
    total_ms = ms.value
    value = edges * args.steps / (total_ms * 1e-3)

    # -- per-loop breakdown: the steady-state graph with a timing event between
    #    loops (sequential capture, mean of K replays); eager launches beside it
    graph_loop_s = cp.replay_timed(max(3, args.steps))
    per_loop = {e.loop.name: [t] for e, t in zip(cp.entries, graph_loop_s)}
    eager = {e.loop.name: [] for e in cp.entries}
    for _ in range(max(3, args.steps // 2)):
        for e, t in zip(cp.entries, cp.run(False, True)):
            eager[e.loop.name].append(t)
    loops = {}
    peak, peak_src = peaks_gbs()
    for e in cp.entries:
        t = statistics.mean(per_loop[e.loop.name])
        loops[e.loop.name] = {"ms": round(t * 1e3, 4),
                              "eager_ms": round(statistics.mean(eager[e.loop.name]) * 1e3, 4),
                              "b_alg": e.alg, "useful_bytes": e.useful,
                              "gbs_alg": round(e.alg / t / 1e9, 1),
                              "frac_of_peak": round(e.alg / t / 1e9 / peak, 4),
                              "schedule": e.sched if e.plan.has_writes else "direct",
                              "nb": e.st.nb, "nc": e.st.nc}
    names = [e.loop.name for e in cp.entries]
    flux = [i for i, n in enumerate(names) if "vflux" in n.split("+")]
    dom = cp.entries[flux[0] if flux else max(range(len(names)), key=lambda i: loops[names[i]]["ms"])]
    t_dom = statistics.mean(per_loop[dom.loop.name])
    achieved = dom.alg / t_dom / 1e9
    traffic = None
    tfile = ROOT / "profiles" / "traffic.json"
    if tfile.exists():
        dom_sched = dom.sched if dom.plan.has_writes else "direct"
        traffic = json.loads(tfile.read_text()).get(dom_sched, {}).get(dom.loop.name)

    # -- end to end through the public API with host buffers ---------------------------------
    pin_mesh(mesh)
    ecfg = ml.BackendConfig(device=0, use_graph=True, residency="host",
                            inc_schedule=sched, inc_schedule_table=table)
    first, _last = cp._stream_plan()
    h2d = sum(d.nbytes for ds in first for d in ds) + sum(g.buffer.nbytes for g in cp.globs)
    d2h = sum(d.nbytes for d in cp.written) + sum(g.buffer.nbytes for g in cp.globs)
    for _ in range(max(2, args.warmup // 2)):     # first runs allocate the copy staging buffers
        ml.run_program(prog, mesh, ecfg)
    t0 = time.perf_counter()
    for _ in range(args.steps):
        ml.run_program(prog, mesh, ecfg)
        _ = [g.value for g in cp.globs]
    e2e_s = time.perf_counter() - t0
    e2e = {"value": edges * args.steps / e2e_s, "unit": "edges/s", "h2d_bytes_per_step": h2d,
           "d2h_bytes_per_step": d2h, "ms_per_step": 1e3 * e2e_s / args.steps}
    e2e["pcie"] = pcie_bounds(h2d, d2h)

    scale_base = scaling_base(args) if args.scale_grid and args.workload == "proxy" else None
    cb = cpu_baseline(args) if not args.no_cpu else None
    line = {
        "metric": METRIC, "value": value, "unit": "edges/s", "n_gpus": 1, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": total_ms / args.steps, "higher_is_better": True,
        "scaling": "strong", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic (jittered 3-D grid, random numbering then CM renumbering)",
        "config": {"workload": wname, "nodes": mesh.sets["nodes"].size, "edges": edges,
                   "loops_per_step": len(prog), "block_size": cfg.block_size,
                   "inc_schedule": args.inc_schedule,
                   "inc_schedule_table": table,
                   "l2": "inputs > 126 MB L2 (no flush needed)",
                   "timing": "CUDA graph replays back to back, CUDA events on the library stream",
                   "parallelism": "single GPU", "device": info["name"], "setup": setup},
        "gpu_launches": cp.launches_per_run() * args.steps,
        "clocks": clk.summary(),
        "roofline": {"bound": "hbm", "kernel": dom.loop.name, "achieved": round(achieved, 1),
                     "peak": peak, "unit": "GB/s", "frac": round(achieved / peak, 4),
                     "traffic": traffic, "peak_source": peak_src,
                     "algorithmic_bytes_per_launch": dom.alg,
                     "spec_peak_gbs": 8000.0,
                     "iteration": {"b_alg": sum(e.alg for e in cp.entries),
                                   "achieved": round(sum(e.alg for e in cp.entries) / (total_ms * 1e-3 / args.steps) / 1e9, 1),
                                   "frac": round(sum(e.alg for e in cp.entries) / (total_ms * 1e-3 / args.steps) / 1e9 / peak, 4)},
                     "mean_loop_ms": round(t_dom * 1e3, 4)},
        "loops": loops,
        "eager_ms_per_step": round(sum(v["eager_ms"] for v in loops.values()), 4),
        "graph_loops_ms_per_step": round(sum(v["ms"] for v in loops.values()), 4),
        "e2e": e2e,
        "cpu_baseline": cb,
        "scaling_base": scale_base,
    }
    print(json.dumps(line))


def _free_port() -> int:
    import socket
    with socket.socket() as sk:
        sk.bind(("127.0.0.1", 0))
        return sk.getsockname()[1]


def self_launch(n: int) -> int:
    """``--gpus N`` without torchrun: start N rank processes of this script
    (RANK/LOCAL_RANK = GPU index, rendezvous on 127.0.0.1 — the reference's
    ``run_ranks`` needs no launcher either, executor.py:690-695).  Rank 0's
    stdout is the bench line; the others are silenced.  The first rank to fail
    stops the rest; the exit code is the first non-zero one."""
    import subprocess
    port = _free_port()
    procs = []
    for r in range(n):
        env = dict(os.environ, RANK=str(r), LOCAL_RANK=str(r), WORLD_SIZE=str(n),
                   LOCAL_WORLD_SIZE=str(n), MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
        procs.append(subprocess.Popen([sys.executable, str(Path(__file__).resolve()), *sys.argv[1:]],
                                      env=env, stdout=None if r == 0 else subprocess.DEVNULL))
    rc = 0
    live = list(procs)
    while live:
        for p in list(live):
            code = p.poll()
            if code is None:
                continue
            live.remove(p)
            if code != 0 and rc == 0:
                rc = code
                for q in live:
                    q.terminate()
        time.sleep(0.05)
    return rc


def launch_probe(args) -> None:
    """``--launch-probe``: each rank joins a gloo group and all-reduces its rank;
    rank 0 prints one JSON line (tests the launcher without a GPU)."""
    import torch
    import torch.distributed as dist
    rank = int(os.environ.get("RANK", "0"))
    if args.launch_probe_fail == rank:
        sys.exit(3)
    dist.init_process_group("gloo")
    t = torch.tensor([rank + 1.0])
    dist.all_reduce(t)
    if rank == 0:
        print(json.dumps({"probe": "ok", "world": dist.get_world_size(), "sum": float(t.item())}))
    dist.destroy_process_group()


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--workload", choices=["proxy", "diffusion"], default="proxy")
    ap.add_argument("--grid", type=int, default=None)
    ap.add_argument("--cpu-grid", type=int, default=None)
    ap.add_argument("--inc-schedule", default="tuned",
                    choices=["tuned", "auto", "gather", "pfold", "colour"])
    ap.add_argument("--schedule-table", default=None,
                    help="per-loop INC schedules, e.g. vflux=pfold,iflux=gather (skips tuning)")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--cpu-sample-only", action="store_true",
                    help="cpu_baseline: time the serial mode on the sample too (not the full workload)")
    ap.add_argument("--scale-grid", type=int, default=139,
                    help="N=1: also time this grid through the multi-GPU executor at world size 1 "
                         "(the base of the 2/4/8-GPU curve); 0 skips it")
    ap.add_argument("--launch-probe", action="store_true", help=argparse.SUPPRESS)
    ap.add_argument("--launch-probe-fail", type=int, default=-1, help=argparse.SUPPRESS)
    args = ap.parse_args()
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ and args.impl == "ours":
        sys.exit(self_launch(args.gpus))
    if args.launch_probe:
        launch_probe(args)
        return
    if args.grid is None:
        # N>1: BASELINE configs[3], the ~8M-edge mesh (139^3 = 7,998,894 edges)
        multi = args.gpus > 1 or int(os.environ.get("WORLD_SIZE", "1")) > 1
        args.grid = (139 if multi else 94) if args.workload == "proxy" else (1633 if multi else 913)
    if args.cpu_grid is None:          # ~2-3 s of CPU per reference-arm step / sampled mode
        if args.impl == "reference":
            args.cpu_grid = 30 if args.workload == "proxy" else 200
        else:
            args.cpu_grid = 24 if args.workload == "proxy" else 160
    if args.impl == "reference":
        run_reference(args)
    else:
        run_ours(args)


if __name__ == "__main__":
    main()
