"""Measurement helpers shared by bench.py and the multi-GPU bench path.

* ``build_workload`` — the benchmark program: the Hydra-shaped proxy
  iteration on a jittered 3-D grid (default 94^3 = 2,465,244 edges, the
  Rotor37 size), numbered randomly then Cuthill–McKee renumbered; or one
  diffusion step on ``gen_mesh``.
* ``clock_sampler`` — ``nvidia-smi`` SM clocks and throttle reasons sampled
  during a timed region.
* ``peaks_gbs`` — the HBM roofline denominator (MEASURED_PEAKS.json, else
  the profiling guide's fallback).
"""
from __future__ import annotations

import json
import os
import statistics
import subprocess
import threading
import time
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent
FALLBACK_PEAK_GBS = 6650.0

__all__ = ["stdout_to_stderr", "build_workload", "clock_sampler", "peaks_gbs", "ClockSampler", "load_reference",
           "cpu_model", "time_reference", "reference_modes"]


def peaks_gbs() -> tuple[float, str]:
    p = ROOT / "MEASURED_PEAKS.json"
    if p.exists():
        try:
            return float(json.loads(p.read_text())["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)"
        except (ValueError, KeyError):
            pass
    return FALLBACK_PEAK_GBS, "fallback (B200_PROFILING.md)"


class ClockSampler:
    """nvidia-smi sampling of SM clocks and throttle reasons (context manager)."""

    FIELDS = ("clocks.sm,clocks.max.sm,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int):
        self.index = index
        self.proc = None
        self.lines: list[str] = []

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--id={self.index}", f"--query-gpu={self.FIELDS}",
                 "--format=csv,noheader,nounits", "-lms", "20"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.thread = threading.Thread(target=self._read, daemon=True)
            self.thread.start()
        except FileNotFoundError:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def __exit__(self, *exc):
        if self.proc is not None:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except subprocess.TimeoutExpired:
                self.proc.kill()

    def summary(self) -> dict:
        sm, mx, reasons = [], [], set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for line in self.lines:
            parts = [p.strip() for p in line.split(",")]
            if len(parts) < 7:
                continue
            try:
                sm.append(float(parts[0]))
                mx.append(float(parts[1]))
            except ValueError:
                continue
            for nm, v in zip(names, parts[3:7]):
                if v.lower() == "active":
                    reasons.add(nm)
        return {"sm_mhz": statistics.median(sm) if sm else None,
                "sm_max_mhz": max(mx) if mx else None, "reasons": sorted(reasons),
                "samples": len(sm)}


def clock_sampler(index: int) -> ClockSampler:
    return ClockSampler(index)


def workload_name(args) -> str:
    """``config.workload`` of a bench line (both arms)."""
    if args.workload == "proxy":
        return f"hydra-proxy iteration, 3-D grid {args.grid}^3"
    return f"diffusion step, gen_mesh({args.grid})"


def build_workload(args):
    """(mesh, program, handles, name, setup timings) for ``args.workload`` / ``args.grid``."""
    from . import apps
    from .renumber import renumber_mesh
    t0 = time.perf_counter()
    if args.workload == "proxy":
        mesh = apps.gen_hex_mesh(args.grid, seed=0)
        apps.shuffle_mesh(mesh, seed=1)
        prog, h = apps.build_hydra_proxy(mesh, steps=1, seed=0)
        name = workload_name(args)
    else:
        mesh = apps.gen_mesh(args.grid)
        apps.shuffle_mesh(mesh, seed=1)
        prog, h = apps.build_diffusion(mesh, steps=1, dtype="float64")
        name = workload_name(args)
    t_gen = time.perf_counter() - t0
    t0 = time.perf_counter()
    renumber_mesh(mesh)
    t_ren = time.perf_counter() - t0
    return mesh, prog, h, name, {"generate_s": round(t_gen, 3), "renumber_s": round(t_ren, 3)}


# -- the stock reference on the host CPU (bench.py's cpu_baseline and reference arm) ------

def load_reference():
    """The stock reference package ``meshloop``: the driver's offline install in
    ``baseline/_ref`` (it travels to the GPU box), else an importable one; None
    if absent.  This is the reference itself, not a restatement."""
    import importlib
    import sys
    p = ROOT / "baseline" / "_ref"
    if (p / "meshloop" / "__init__.py").exists() and str(p) not in sys.path:
        sys.path.append(str(p))
    try:
        return importlib.import_module("meshloop")
    except ImportError:
        return None


def cpu_model() -> str:
    """``lscpu`` model name of this host."""
    try:
        out = subprocess.run(["lscpu"], capture_output=True, text=True, timeout=10).stdout
        for line in out.splitlines():
            if line.startswith("Model name:"):
                return line.split(":", 1)[1].strip()
    except (OSError, subprocess.SubprocessError):
        pass
    try:
        for line in Path("/proc/cpuinfo").read_text().splitlines():
            if line.startswith("model name"):
                return line.split(":", 1)[1].strip()
    except OSError:
        pass
    return "unknown"


def reference_modes(cores: int) -> dict:
    """The reference's CPU execution modes (executor.py:707-729) with all host
    threads: serial, threads (nthreads = cores), ranks (largest power of two
    <= cores, RCB on the ``coords`` dat: partition.py:81-106)."""
    p = 1
    while p * 2 <= cores:
        p *= 2
    return {"serial": {}, "threads": {"backend": "threads", "nthreads": cores},
            "ranks": {"backend": "ranks", "nranks": p, "partitioner": "rcb"}}


def _split_at_reduced_reads(program):
    """Programs to run one after another so that a global a loop reduces is
    final before a later loop READs it.  The reference's ranks backend folds
    reductions only when the whole program ends (executor.py:653-660), so one
    call over the proxy iteration would hand ``update`` the initial +inf of
    ``dt_min``; splitting after ``dt_calc`` keeps its arithmetic finite."""
    parts, cur, reduced = [], [], set()
    for l in program:
        reads = {id(a.glob) for a in l.args if a.kind == "global" and a.mode.name == "READ"}
        if reads & reduced and cur:
            parts.append(cur)
            cur, reduced = [], set()
        cur.append(l)
        reduced |= {id(a.glob) for a in l.args if a.kind == "global" and a.mode.name != "READ"}
    if cur:
        parts.append(cur)
    return parts


def time_reference(R, mesh, prog, mode: str, cores: int, runs: int = 1, warm: int = 0):
    """Seconds per stock ``meshloop.run_program`` call of ``prog`` (exported to
    reference objects) in ``mode``; ``warm`` untimed calls first (the threads
    backend builds and caches its plans on the first call).  Returns
    (seconds per run, number of run_program calls per run)."""
    from .foreign import export_mesh, export_program
    ref = export_mesh(mesh, R)
    rprog = export_program(prog, ref, R)
    cfg = R.BackendConfig(**reference_modes(cores)[mode])
    parts = _split_at_reduced_reads(rprog) if mode == "ranks" else [rprog]
    for _ in range(warm):
        for p in parts:
            R.run_program(p, ref, cfg)
    t0 = time.perf_counter()
    for _ in range(runs):
        for p in parts:
            R.run_program(p, ref, cfg)
    return (time.perf_counter() - t0) / runs, len(parts)


class stdout_to_stderr:
    """Route file descriptor 1 to stderr for the duration (NCCL and other
    native libraries print banners on stdout, which must carry only the one
    JSON bench line); ``write_line`` prints to the real stdout meanwhile."""

    def __enter__(self):
        import sys
        sys.stdout.flush()
        self.saved = os.dup(1)
        os.dup2(2, 1)
        return self

    def write_line(self, text: str) -> None:
        os.write(self.saved, (text + "\n").encode())

    def __exit__(self, *exc):
        import sys
        sys.stdout.flush()
        os.dup2(self.saved, 1)
        os.close(self.saved)
