"""Set up the benchmark workload and run it eagerly (ncu captures, schedule /
layout / block-size sweeps).

    python scripts/profile_proxy.py [--grid 94] [--iters 3] [--block-size 256 128]
                                    [--inc-schedule gather pfold colour] [--soa 4]
"""
import argparse
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))

import paper_1403_7209_b200 as ml                  # noqa: E402
from paper_1403_7209_b200 import apps              # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--grid", type=int, default=94)
ap.add_argument("--iters", type=int, default=3)
ap.add_argument("--block-size", type=int, nargs="+", default=[256])
ap.add_argument("--soa", type=int, default=4, help="auto-SOA threshold; -1 = all AOS")
ap.add_argument("--inc-schedule", nargs="+", default=["gather"])
ap.add_argument("--no-renumber", action="store_true")
ap.add_argument("--kd", type=int, default=0, help="k-d leaf size: renumber nodes in k-d order after CM")
ap.add_argument("--chain", type=int, nargs="+", default=[1], help="loop chaining on/off")
ap.add_argument("--aos-dats", nargs="*", default=[], help="dats switched to AoS after generation")

args = ap.parse_args()
mesh = apps.gen_hex_mesh(args.grid, seed=0, auto_soa_threshold=None if args.soa < 0 else args.soa)
apps.shuffle_mesh(mesh, seed=1)
prog, h = apps.build_hydra_proxy(mesh, steps=1, seed=0)
if not args.no_renumber:
    ml.renumber_mesh(mesh)
for name in args.aos_dats:
    from paper_1403_7209_b200.core import AOS, transform_layout
    transform_layout(mesh.dats[name], AOS)
if args.kd:
    import numpy as np
    from paper_1403_7209_b200.renumber import Permutation, apply_permutation, row_order_by_targets, _forward

    def kd_order(xyz, leaf):
        out, stack = [], [np.arange(len(xyz))]
        while stack:
            a = stack.pop()
            if len(a) <= leaf:
                out.append(np.sort(a))
                continue
            p = xyz[a]
            ax = int(np.argmax(p.max(0) - p.min(0)))
            o = np.lexsort((a, p[:, ax]))
            m = (len(a) + 1) // 2
            stack.append(a[o[m:]])
            stack.append(a[o[:m]])
        return np.concatenate(out)
    order = kd_order(mesh.dats["coords"].fetch(), args.kd)
    apply_permutation(mesh, Permutation("nodes", _forward(order), order, mesh.version))
    for sname in ("edges", "bedges"):
        m = next(m for m in mesh.maps.values() if m.from_set.name == sname)
        apply_permutation(mesh, row_order_by_targets(mesh, m))
import itertools
import statistics
for bs, ch in itertools.product(args.block_size, args.chain):
    for sched in args.inc_schedule:
        cfg = ml.BackendConfig(device=0, block_size=bs, inc_schedule=sched, chain_loops=bool(ch))
        per = {}
        for i in range(args.iters):
            r = ml.run_program(prog, mesh, cfg)
            if i == 0 and args.iters > 1:
                continue                                   # compile + upload
            for p in r.perf:
                per.setdefault(p.loop, []).append((p.time_sec, p.gb_per_sec_alg))
        med = {k: (statistics.median(t for t, _ in v), statistics.median(g for _, g in v)) for k, v in per.items()}
        tot = sum(t for t, _ in med.values())
        print(f"[{sched} kd={args.kd} bs={bs} soa={args.soa} chain={ch}] "
              f"total={tot*1e3:.3f}ms " +
              " ".join(f"{k}={t*1e3:.3f}ms/{g:.0f}GBs" for k, (t, g) in med.items()), flush=True)
