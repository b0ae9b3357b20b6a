"""e2e probe (not product code): where the host-residency step's time goes.

Builds the bench workload (94^3 proxy), then times, per step: the public
run_program(residency="host") call; its H2D copies alone (the streamed
plan's inputs, same copy calls); its D2H copies alone; one 1-D copy of the
same byte count; and the compute alone (graph replay).

    python scripts/e2e_probe.py [--steps 10]
"""
import argparse
import json
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))

import paper_1403_7209_b200 as ml                      # noqa: E402
from paper_1403_7209_b200 import _native as N          # noqa: E402
from paper_1403_7209_b200.bench_support import build_workload   # noqa: E402
from paper_1403_7209_b200.device import dat_mirror, pin_mesh     # noqa: E402
from paper_1403_7209_b200.executor import compile_program        # noqa: E402


def wall(fn, steps):
    fn()
    N.check(N.lib().ml_sync_all())
    t0 = time.perf_counter()
    for _ in range(steps):
        fn()
    N.check(N.lib().ml_sync_all())
    return (time.perf_counter() - t0) / steps * 1e3


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--steps", type=int, default=10)
    a = ap.parse_args()
    args = argparse.Namespace(workload="proxy", grid=94)
    mesh, prog, _h, _name, _ = build_workload(args)
    N.init(0)
    pin_mesh(mesh)
    cfg = ml.BackendConfig(device=0, use_graph=True, residency="host")
    ml.run_program(prog, mesh, cfg)
    cp = compile_program(prog, mesh, cfg)
    first, last = cp._stream_plan()
    ins = [d for ds in first for d in ds]
    outs = [d for ds in last for d in ds]
    L = N.lib()
    out = {"h2d_bytes": sum(d.nbytes for d in ins), "d2h_bytes": sum(d.nbytes for d in outs)}
    out["run_program_ms"] = wall(lambda: ml.run_program(prog, mesh, cfg), a.steps)

    def h2d():
        for d in ins:
            d._dev.copy_h2d(d._host)
    out["h2d_only_ms"] = wall(h2d, a.steps)

    def d2h():
        for d in outs:
            d._dev.copy_d2h(d._host)
    out["d2h_only_ms"] = wall(d2h, a.steps)

    def both():
        h2d()
        d2h()
    out["h2d_and_d2h_concurrent_ms"] = wall(both, a.steps)
    big = N.PinnedArray((out["h2d_bytes"],), "uint8")
    dev = N.DeviceBuffer(out["h2d_bytes"])
    out["h2d_1d_same_bytes_ms"] = wall(lambda: N.check(L.ml_copy_h2d(dev.ptr, N.ptr(big.array),
                                                                    out["h2d_bytes"])), a.steps)
    dcfg = ml.BackendConfig(device=0, use_graph=True)
    for d in mesh.dats.values():
        dat_mirror(d)
    ml.run_program(prog, mesh, dcfg)
    dcp = compile_program(prog, mesh, dcfg)
    out["compute_replay_ms"] = wall(lambda: dcp.replay(1), a.steps)
    out["run_streamed_only_ms"] = wall(cp.run_streamed, a.steps)
    print(json.dumps({k: (round(v, 3) if isinstance(v, float) else v) for k, v in out.items()}))


if __name__ == "__main__":
    main()
