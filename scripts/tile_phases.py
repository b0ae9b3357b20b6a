"""Per-phase cycle counts of the tile kernel (library built with
MESHLOOP_NVCC_FLAGS=-DML_TILE_PROFILE): staging issue, staging wait, compute +
colour phases, write-back; mean/median over tiles, per edge loop."""
import argparse
import ctypes as C
import sys
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import paper_1403_7209_b200 as ml                  # noqa: E402
from paper_1403_7209_b200 import _native as N, apps  # noqa: E402
from paper_1403_7209_b200.executor import compile_program  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--tile-smem", type=int, default=100)
ap.add_argument("--tile-threads", type=int, default=256)
args = ap.parse_args()
mesh = apps.gen_hex_mesh(94, seed=0)
apps.shuffle_mesh(mesh, seed=1)
prog, h = apps.build_hydra_proxy(mesh, steps=1, seed=0)
ml.renumber_mesh(mesh)
cfg = ml.BackendConfig(device=0, inc_schedule="tile", tile_smem_kb=args.tile_smem, tile_threads=args.tile_threads)
cp = compile_program(prog, mesh, cfg)
cp.run(False, True)
for e in cp.entries:
    if e.tile is None:
        continue
    nt = e.tile.count
    buf = N.DeviceBuffer(nt * 32)
    d = e.desc
    d.fold_buf = buf.ptr
    for _ in range(2):
        N.check(N.lib().ml_loop_run(C.byref(d)))
    N.check(N.lib().ml_synchronize())
    host = np.empty(nt * 4, np.int64)
    buf.download(host)
    host = host.reshape(nt, 4)
    d.fold_buf = None
    tot = host.sum(1)
    print(f"{e.loop.name}: tiles={nt} cycles/tile mean={tot.mean():.0f} "
          f"[issue {host[:,0].mean():.0f} | wait {host[:,1].mean():.0f} | compute+phases {host[:,2].mean():.0f} "
          f"| writeback {host[:,3].mean():.0f}]  median total {np.median(tot):.0f}")
