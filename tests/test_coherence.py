"""Host/device coherence across runs (GPU).

* A compiled program bakes each dat's layout into its loop descriptors; a
  ``transform_layout`` between runs must invalidate it (the reference reads
  ``d.layout`` on every run, core.py:179-192 / executor.py:149-160).
* A device-resident run leaves written dats newer on the device; a following
  host-residency run (streamed or not) must not overwrite them with the
  stale host payload.
"""
from __future__ import annotations

import numpy as np
import pytest

import paper_1403_7209_b200 as ml
from paper_1403_7209_b200 import apps
from oracle import bulk


def _proxy(N=9, seed=3):
    mesh = apps.gen_hex_mesh(N, seed=seed)
    prog, h = apps.build_hydra_proxy(mesh, steps=1, seed=seed)
    return mesh, prog, h


def _close(a, b):
    np.testing.assert_allclose(a, b, rtol=1e-12, atol=1e-12 * max(np.abs(b).max(), 1e-300))


@pytest.mark.gpu
@pytest.mark.parametrize("use_graph", [False, True])
def test_transform_layout_between_runs(use_graph):
    mesh, prog, h = _proxy()
    ref, rprog, rh = _proxy()
    cfg = ml.BackendConfig(use_graph=use_graph)
    ml.run_program(prog, mesh, cfg)
    bulk.run_program(rprog)
    for name in ("q", "aux", "grad"):
        target = ml.AOS if mesh.dats[name].layout is ml.SOA else ml.SOA
        ml.transform_layout(mesh.dats[name], target)
        ml.transform_layout(ref.dats[name], target)
    ml.run_program(prog, mesh, cfg)
    bulk.run_program(rprog)
    for k in ("q", "q_old", "res", "grad", "dt_loc"):
        _close(h[k].fetch(), rh[k].fetch())


@pytest.mark.gpu
@pytest.mark.parametrize("host_mode", ["streamed", "eager"])
def test_device_then_host_residency_keeps_device_results(host_mode):
    mesh, prog, h = _proxy()
    ref, rprog, rh = _proxy()
    ml.run_program(prog, mesh, ml.BackendConfig())                 # device-resident
    bulk.run_program(rprog)
    hcfg = (ml.BackendConfig(residency="host", use_graph=True) if host_mode == "streamed"
            else ml.BackendConfig(residency="host"))
    ml.run_program(prog, mesh, hcfg)
    bulk.run_program(rprog)
    for k in ("q", "q_old", "res", "grad", "dt_loc"):
        _close(h[k].fetch(), rh[k].fetch())
    # and back to device residency after a host write
    mesh.dats["q"].data[:5] += 1.0
    ref.dats["q"].data[:5] += 1.0
    ml.run_program(prog, mesh, ml.BackendConfig())
    bulk.run_program(rprog)
    for k in ("q", "q_old", "res", "grad", "dt_loc"):
        _close(h[k].fetch(), rh[k].fetch())


@pytest.mark.gpu
@pytest.mark.parametrize("n", [1, 63, 64, 65, 4097, 10000])
@pytest.mark.parametrize("dim", [6, 8, 19])
def test_soa_device_copies_round_trip(n, dim):
    """SOA dats of dim ML_SEG_MIN_DIM.. live on the device in blocks of
    2^ML_SEG_SHIFT elements (device.py segmented(); host copies repacked on
    the device, ml_seg_copy), narrower ones as pitched rows: host -> device ->
    host is exact for ragged set sizes, a direct loop moves the right
    components, and streamed (H2D/D2H stream) copies agree."""
    from paper_1403_7209_b200 import _native as N
    from paper_1403_7209_b200.device import dat_mirror, segmented
    rng = np.random.default_rng(n * 31 + dim)
    mesh = ml.Mesh()
    nodes = mesh.decl_set("nodes", n)
    vals = rng.random((n, dim))
    q = mesh.decl_dat("q", nodes, dim, "float64", vals.ravel())
    q_old = mesh.decl_dat("q_old", nodes, dim, "float64", np.zeros(n * dim))
    assert q.layout is ml.SOA
    assert segmented(q) == (dim >= 8)
    m = dat_mirror(q)
    back = np.empty_like(q._host)
    m.download(back)
    np.testing.assert_array_equal(back, q._host)
    if dim == 6:                                   # proxy_save: a direct loop over the rows
        ml.run_program([ml.Loop("save", nodes, [ml.arg_direct(q, ml.READ), ml.arg_direct(q_old, ml.WRITE)],
                                apps._k_proxy_save)], mesh, ml.BackendConfig())
        np.testing.assert_array_equal(q_old.fetch(), vals)
    host2 = np.ascontiguousarray(rng.random(q._host.shape))
    m.copy_h2d(host2)                              # streamed: H2D stream, then D2H stream
    N.check(N.lib().ml_sync_all())
    out = np.empty_like(host2)
    m.copy_d2h(out)
    N.check(N.lib().ml_sync_all())
    np.testing.assert_array_equal(out, host2)


@pytest.mark.gpu
def test_pinned_host_residency_matches_oracle():
    """bench.py's e2e path: payloads re-homed in pinned memory (pin_mesh), so
    segmented dats go down through the repack kernel writing the host buffer
    directly and up through the double-staged H2D path; two streamed
    host-residency iterations match the oracle."""
    from paper_1403_7209_b200.device import pin_mesh
    mesh, prog, h = _proxy(N=14, seed=8)
    ref, rprog, rh = _proxy(N=14, seed=8)
    pin_mesh(mesh, min_bytes=1)
    cfg = ml.BackendConfig(residency="host", use_graph=True)
    for _ in range(2):
        ml.run_program(prog, mesh, cfg)
        bulk.run_program(rprog)
    for k in ("q", "q_old", "res", "grad", "dt_loc"):
        _close(h[k].fetch(), rh[k].fetch())
    for k in ("lim", "aux"):                      # read-only segmented dats survive the round trips
        np.testing.assert_array_equal(mesh.dats[k].fetch(), ref.dats[k].fetch())


@pytest.mark.gpu
def test_record_columns_fall_back_when_a_loop_differs():
    """grad_edge with its q arguments' map slots swapped: the loop's record
    columns no longer match the functor's declaration, so the generic kernel
    (columns from the launch parameters) runs — and matches the oracle; the
    stock loop takes the compile-time-column kernel."""
    from paper_1403_7209_b200.core import READ, Loop, arg_indirect
    from paper_1403_7209_b200.executor import compile_program
    mesh, prog, h = _proxy(N=10, seed=9)
    ref, rprog, rh = _proxy(N=10, seed=9)

    def swap(p, hh):
        g = p[2]
        args = list(g.args)
        args[1] = arg_indirect(hh["q"], args[1].map, 2, READ)
        args[2] = arg_indirect(hh["q"], args[2].map, 1, READ)
        return p[:2] + [Loop(g.name, g.iter_set, args, g.kernel)]
    cfg = ml.BackendConfig(inc_schedule="gather")
    assert compile_program(prog[:3], mesh, cfg).entries[-1].desc.rec_fixed == 1
    p3, r3 = swap(prog, h), swap(rprog, rh)
    assert compile_program(p3, mesh, cfg).entries[-1].desc.rec_fixed == 0
    ml.run_program(p3, mesh, cfg)
    bulk.run_program(r3)
    np.testing.assert_array_equal(h["grad"].fetch(), rh["grad"].fetch())
