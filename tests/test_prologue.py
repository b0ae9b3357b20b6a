"""Cross-set prologues (ML_REGISTER_PROLOGUE, executor._link_prologues): the
proxy's save+dt_calc (direct over nodes) runs inside grad_edge's gather
kernel over nodes.  Nothing about the arithmetic changes — the direct part is
per element, the MIN is exact, the gather keeps serial order — so results are
bitwise the unlinked ones and the oracle's, in every run mode."""
from __future__ import annotations

import numpy as np
import pytest

import paper_1403_7209_b200 as ml
from paper_1403_7209_b200 import apps
from paper_1403_7209_b200.core import READ, Loop, arg_indirect
from oracle import bulk

pytestmark = pytest.mark.gpu


def _proxy(N=12, seed=4, steps=1):
    mesh = apps.gen_hex_mesh(N, seed=seed)
    apps.shuffle_mesh(mesh, seed=seed + 1)
    prog, h = apps.build_hydra_proxy(mesh, steps=steps, seed=seed)
    ml.renumber_mesh(mesh)
    return mesh, prog, h


KEYS = ("q", "q_old", "grad", "res", "dt_loc")


@pytest.mark.parametrize("mode", [{}, {"use_graph": True}, {"residency": "host", "use_graph": True},
                                  {"residency": "host"}, {"time_loops": False}])
def test_save_dt_runs_inside_grad_edge_bitwise(mode):
    from paper_1403_7209_b200.executor import compile_program
    mesh, prog, h = _proxy()
    rmesh, rprog, rh = _proxy()
    cfg = ml.BackendConfig(**mode)
    cp = compile_program(prog, mesh, cfg)
    assert [n for n, _ in cp.run_names()] == ["save+dt_calc+grad_edge", "iflux+vflux", "update", "bc"]
    assert cp.absorbed == [True, False, False, False, False]
    # save+dt_calc+grad_edge 1, iflux+vflux 2 (pfold passes), update 1, bc 1
    assert cp.launches_per_run() == 5
    ml.run_program(prog[:3], mesh, cfg)           # save, dt_calc, grad_edge
    bulk.run_program(rprog[:3])
    for k in ("q_old", "dt_loc", "grad"):
        np.testing.assert_array_equal(h[k].fetch(), rh[k].fetch(), err_msg=k)
    assert h["dt_min"][0].value == rh["dt_min"][0].value
    res = ml.run_program(prog, mesh, cfg)         # the whole iteration
    bulk.run_program(rprog)
    if not mode:                                  # eager timed run: one record for the pair
        assert "save+dt_calc+grad_edge" in [r.loop for r in res.perf]
    for k in KEYS:
        np.testing.assert_allclose(h[k].fetch(), rh[k].fetch(), rtol=1e-12, atol=1e-12, err_msg=k)
    assert h["dt_min"][0].value == rh["dt_min"][0].value


def test_linked_equals_unlinked_bitwise():
    mesh, prog, h = _proxy(seed=7, steps=2)
    mesh2, prog2, h2 = _proxy(seed=7, steps=2)
    ml.run_program(prog, mesh, ml.BackendConfig(use_graph=True))
    off = ml.BackendConfig(use_graph=True, prologue_loops=False)
    ml.run_program(prog2, mesh2, off)
    from paper_1403_7209_b200.executor import compile_program
    assert not any(compile_program(prog2, mesh2, off).absorbed)
    tab = ml.BackendConfig(use_graph=True, inc_schedule_table={"grad_edge": "gather", "iflux+vflux": "pfold"})
    assert compile_program(prog, mesh, tab).absorbed[0]          # a table choosing gather keeps the link
    for k in KEYS:
        np.testing.assert_array_equal(h[k].fetch(), h2[k].fetch(), err_msg=k)
    for a, b in zip(h["dt_min"], h2["dt_min"]):
        assert a.value == b.value


def test_hazard_keeps_loops_apart():
    """grad_edge reading the dat save writes: linking would let a thread read a
    neighbour's row before the prologue wrote it, so the loops stay apart."""
    from paper_1403_7209_b200.executor import compile_program
    mesh, prog, h = _proxy()
    rmesh, rprog, rh = _proxy()

    def rewire(p, hh):
        g = p[2]
        args = list(g.args)
        args[1] = arg_indirect(hh["q_old"], args[1].map, args[1].slot + 1, READ)
        args[2] = arg_indirect(hh["q_old"], args[2].map, args[2].slot + 1, READ)
        return p[:2] + [Loop(g.name, g.iter_set, args, g.kernel)]
    prog3, rprog3 = rewire(prog, h), rewire(rprog, rh)
    cp = compile_program(prog3, mesh, ml.BackendConfig())
    assert not any(cp.absorbed)
    ml.run_program(prog3, mesh, ml.BackendConfig())
    bulk.run_program(rprog3)
    np.testing.assert_array_equal(h["grad"].fetch(), rh["grad"].fetch())
