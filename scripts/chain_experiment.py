"""Loop-chaining experiment: iflux + vflux as one loop (functor proxy_fluxes)."""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import paper_1403_7209_b200 as ml                  # noqa: E402
from paper_1403_7209_b200 import apps              # noqa: E402
from paper_1403_7209_b200.kernels import device_kernel  # noqa: E402

mesh = apps.gen_hex_mesh(94, seed=0)
apps.shuffle_mesh(mesh, seed=1)
prog, h = apps.build_hydra_proxy(mesh, steps=1, seed=0)
ml.renumber_mesh(mesh)
names = [l.name for l in prog]
i, v = names.index("iflux"), names.index("vflux")
li, lv = prog[i], prog[v]


@device_kernel("proxy_fluxes")
def fluxes(*a):
    pass


args = list(li.args[:7]) + [lv.args[3], lv.args[4], lv.args[7], lv.args[8]] + list(li.args[7:9])
fused = ml.Loop("fluxes", li.iter_set, args, fluxes)
chained = prog[:i] + [fused] + prog[v + 1:]
for sched in ("gather", "pfold"):
    for label, p in (("separate", prog), ("chained", chained)):
        cfg = ml.BackendConfig(device=0, inc_schedule=sched)
        for _ in range(4):
            r = ml.run_program(p, mesh, cfg)
        tot = sum(x.time_sec for x in r.perf)
        print(f"[{sched} {label}] total={tot*1e3:.3f}ms " +
              " ".join(f"{x.loop}={x.time_sec*1e3:.3f}" for x in r.perf), flush=True)
