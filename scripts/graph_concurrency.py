"""Graph replay time of the 94^3 proxy iteration with and without concurrent
loop lanes (ml_program DAG); 200 replays timed with CUDA events."""
import sys, time, ctypes as C
sys.path.insert(0, "/root/repo")
import paper_1403_7209_b200 as ml
from paper_1403_7209_b200 import apps, _native as N
from paper_1403_7209_b200.executor import compile_program
mesh = apps.gen_hex_mesh(94, seed=0); apps.shuffle_mesh(mesh, seed=1)
prog, h = apps.build_hydra_proxy(mesh, steps=1, seed=0); ml.renumber_mesh(mesh)
for conc in (True, False, True, False):
    cfg = ml.BackendConfig(device=0, use_graph=True, concurrent_loops=conc)
    cp = compile_program(prog, mesh, cfg)
    cp.replay(20)
    timer = C.c_void_p(); N.check(N.lib().ml_timer_create(C.byref(timer)))
    ms = C.c_float()
    N.check(N.lib().ml_synchronize()); N.check(N.lib().ml_timer_start(timer))
    cp.replay(200)
    N.check(N.lib().ml_timer_stop(timer, C.byref(ms)))
    print("concurrent", conc, round(ms.value / 200, 4), "ms/step", flush=True)
