"""Programs built from the stock reference package's own objects.

North_star: Hydra-style solver code written against ``meshloop`` runs
unchanged.  These tests build programs with the reference's ``Mesh`` /
``Dat`` / ``Loop`` classes and its own app builders (``meshloop.apps``,
reference ``apps.py:159-304``), run them on B200 through

* the reference's own ``meshloop.run_program`` with
  ``BackendConfig(backend="cuda")`` after :func:`foreign.install`, and
* the branch INTEGRATION.md shows (``b200.run_program(program, ref_mesh,
  b200.BackendConfig(...))``),

and compare against the stock reference executing the same program on the CPU
(``meshloop.run_program(program, mesh, BackendConfig())``, the serial
backend, executor.py:711-715) or — at BASELINE sizes where the reference
would take minutes — against the vectorised oracle (``oracle/bulk.py``,
pinned bit-for-bit to the reference on the golden cases).

Bars: int64 bit-exact; float64 ``rtol=1e-12`` (reference
``test_acceptance.py:94-97``) with an absolute floor of ``1e-12·max|ref|``
for raw INC accumulators whose cancelling sums the schedule reorders.
"""
from __future__ import annotations

import numpy as np
import pytest

import paper_1403_7209_b200 as b
from paper_1403_7209_b200 import apps, foreign
from oracle import bulk


def _close(got, want, what=""):
    want = np.asarray(want)
    if want.dtype.kind in "iu":
        np.testing.assert_array_equal(got, want, what)
        return
    floor = 1e-12 * float(np.max(np.abs(want))) if want.size else 0.0
    np.testing.assert_allclose(got, want, rtol=1e-12, atol=floor, err_msg=what)


def _globs(program):
    out = []
    for l in program:
        for a in l.args:
            if a.kind == "global" and all(a.glob is not g for g in out):
                out.append(a.glob)
    return out


# -- CPU: the adoption layer itself ------------------------------------------------------

def test_shadow_shares_reference_arrays(R):
    m = R.apps.gen_mesh(6)
    prog, h = R.apps.build_diffusion(m, 2, dtype="int64")
    sh = foreign.shadow_mesh(m)
    loops, globs = sh.translate(m, prog)
    assert [l.name for l in loops] == [l.name for l in prog]
    for name, rd in m.dats.items():
        assert sh.mesh.dats[name]._host is rd.data
        assert sh.mesh.dats[name].layout.name == rd.layout.name
    for name, rm in m.maps.items():
        assert sh.mesh.maps[name].table is rm.table
    # one shadow Global per reference Global, sharing its buffer
    assert len(globs) == 2 and all(pg.buffer is rg.buffer for rg, pg in globs)
    assert sh.translate(m, prog)[0] is loops                  # cached per program
    assert foreign.shadow_mesh(m) is sh


def test_shadow_rebinds_replaced_payload_and_renumbering(R):
    m = R.apps.gen_mesh(5)
    prog, _ = R.apps.build_diffusion(m, 1, dtype="int64")
    sh = foreign.shadow_mesh(m)
    sh.translate(m, prog)
    d = m.dats["coords"]
    R.transform_layout(d, R.SOA)              # assigns a new array (core.py:187-190)
    sh.sync_in(m, [])
    assert sh.mesh.dats["coords"]._host is d.data and sh.mesh.dats["coords"].layout is b.SOA
    R.renumber_mesh(m)                        # version bump -> new shadow over the new tables
    sh2 = foreign.shadow_mesh(m)
    assert sh2 is not sh and sh2.mesh.maps["edge_nodes"].table is m.maps["edge_nodes"].table


def test_foreign_objects_rejected_when_not_declared_on_mesh(R):
    m1, m2 = R.apps.gen_mesh(4), R.apps.gen_mesh(4)
    prog, _ = R.apps.build_diffusion(m2, 1, dtype="int64")
    with pytest.raises(b.ExecError, match="not declared on this mesh"):
        foreign.shadow_mesh(m1).translate(m1, prog)


def test_install_adds_cuda_backend_and_keeps_stock_backends(R):
    foreign.install(R)
    foreign.install(R)                                        # idempotent
    assert "cuda" in R.executor._BACKENDS
    cfg = R.BackendConfig(backend="cuda", block_size=64)
    assert foreign.to_backend_config(cfg).block_size == 64
    # the stock serial backend still runs the reference's own code
    m = R.apps.gen_mesh(5)
    prog, h = R.apps.build_diffusion(m, 1, dtype="int64")
    R.run_program(prog, m, R.BackendConfig())
    m2 = R.apps.gen_mesh(5)
    prog2, h2 = R.apps.build_diffusion(m2, 1, dtype="int64")
    R.executor.run_program.__wrapped__(prog2, m2, R.BackendConfig())
    np.testing.assert_array_equal(h["u"].fetch(), h2["u"].fetch())


def test_export_mesh_round_trips_through_reference_declarations(R):
    pm = apps.gen_hex_mesh(5, seed=2)
    for thr in (4, None, 0):
        rm = foreign.export_mesh(pm, R, auto_soa_threshold=thr)
        for n, d in pm.dats.items():
            np.testing.assert_array_equal(rm.dats[n].fetch(), d.fetch())
            want = "SOA" if thr is not None and d.dim > thr else "AOS"
            assert rm.dats[n].layout.name == want
        for n, mp in pm.maps.items():
            np.testing.assert_array_equal(rm.maps[n].table, mp.table)


def test_oracle_resolver_reads_reference_closure_constants(R):
    m = R.apps.gen_mesh(5)
    for dtype in ("float64", "int64"):
        prog, h = R.apps.build_diffusion(m if dtype == "float64" else R.apps.gen_mesh(5), 1, dtype=dtype)
        bnd = bulk.resolve(prog[2].kernel)
        assert bnd.functor == "diffusion_update"
        assert (bnd.fconsts if dtype == "float64" else bnd.iconsts) == prog[2].kernel.__defaults__


# -- GPU: stock reference programs on B200 vs the stock reference on the CPU -------------

def _ref_app(R, app, n, dtype, steps=2):
    m = R.apps.gen_mesh(n)
    if app == "diffusion":
        prog, h = R.apps.build_diffusion(m, steps, dtype=dtype)
        keys = ("u", "flux")
    else:
        prog, h = R.apps.build_cell_area(m, dtype=dtype)
        keys = tuple(k for k, v in h.items() if hasattr(v, "fetch"))
    return m, prog, h, keys


def _compare(R, h_got, h_want, keys, prog_got, prog_want):
    for k in keys:
        _close(h_got[k].fetch(), h_want[k].fetch(), k)
    for g, w in zip(_globs(prog_got), _globs(prog_want)):
        _close(g.buffer, w.buffer, g.name)


@pytest.mark.gpu
@pytest.mark.parametrize("entry", ["install", "integration_branch"])
@pytest.mark.parametrize("app,dtype", [("diffusion", "int64"), ("diffusion", "float64"),
                                       ("cell_area", "int64"), ("cell_area", "float64")])
def test_reference_apps_on_b200_match_stock_reference(R, entry, app, dtype):
    m, prog, h, keys = _ref_app(R, app, 40, dtype)
    mw, progw, hw, _ = _ref_app(R, app, 40, dtype)
    R.run_program(progw, mw, R.BackendConfig())                  # stock serial
    if entry == "install":
        foreign.install(R)
        res = R.run_program(prog, m, R.BackendConfig(backend="cuda"))
    else:
        res = b.run_program(prog, m, b.BackendConfig(block_size=128))
    assert [r.loop for r in res.perf] and m.frozen
    _compare(R, h, hw, keys, prog, progw)


@pytest.mark.gpu
def test_reference_program_repeated_runs_and_host_writes(R):
    """Run, write a dat in place through the reference object, run again: the
    backend must see the host write and leave every result in dat.data."""
    foreign.install(R)
    m, prog, h, keys = _ref_app(R, "diffusion", 30, "int64", steps=1)
    mw, progw, hw, _ = _ref_app(R, "diffusion", 30, "int64", steps=1)
    for it in range(3):
        R.run_program(prog, m, R.BackendConfig(backend="cuda"))
        R.run_program(progw, mw, R.BackendConfig())
        _compare(R, h, hw, keys, prog, progw)
        for mm in (m, mw):
            mm.dats["u"].data[::7] += 3 + it          # in-place host write between runs
    R.transform_layout(m.dats["u"], R.SOA)            # payload replaced: still coherent
    R.transform_layout(mw.dats["u"], R.SOA)
    R.run_program(prog, m, R.BackendConfig(backend="cuda"))
    R.run_program(progw, mw, R.BackendConfig())
    _compare(R, h, hw, keys, prog, progw)


@pytest.mark.gpu
@pytest.mark.parametrize("dtype", ["int64", "float64"])
def test_config1_kuhn47_edge_flux_matches_stock_reference(R, dtype):
    """BASELINE config 1: ~100K-node 3-D mesh (Kuhn grid N=47, 700,534 edges),
    the reference's own diffusion program (edge_flux = apps.py:217-220), B200 vs
    the stock reference's serial run."""
    pm = apps.gen_kuhn_mesh(47, seed=0)
    assert pm.sets["edges"].size == 700534
    m, mw = foreign.export_mesh(pm, R), foreign.export_mesh(pm, R)
    prog, h = R.apps.build_diffusion(m, 1, dtype=dtype)
    progw, hw = R.apps.build_diffusion(mw, 1, dtype=dtype)
    foreign.install(R)
    R.run_program(prog, m, R.BackendConfig(backend="cuda"))
    R.run_program(progw, mw, R.BackendConfig())
    _compare(R, h, hw, ("u", "flux"), prog, progw)


@pytest.mark.gpu
@pytest.mark.parametrize("n", [913, 1633])
def test_reference_f64_diffusion_at_config_b_and_d(R, n):
    """f64 diffusion from the reference's own generator and builder at BASELINE
    config B (gen_mesh(913), 2.50M edges) and D (gen_mesh(1633), 8.0M edges)
    on B200 vs the oracle (the stock serial run would take minutes)."""
    m = R.apps.gen_mesh(n)
    prog, h = R.apps.build_diffusion(m, 2, dtype="float64")
    mw = R.apps.gen_mesh(n)
    progw, hw = R.apps.build_diffusion(mw, 2, dtype="float64")
    b.run_program(prog, m, b.BackendConfig())
    bulk.run_program(progw)
    _compare(R, h, hw, ("u", "flux"), prog, progw)


@pytest.mark.gpu
@pytest.mark.parametrize("renumber", [False, True])
@pytest.mark.parametrize("thr", [4, None, 0])
def test_config3_proxy_layouts_and_renumbering_at_94(R, thr, renumber):
    """BASELINE config 3: the 2.47M-edge proxy iteration with the reference's
    auto-SOA policy at 4 / None (all AOS) / 0 (all SOA), with and without the
    stock reference's renumbering (renumber.py:177-202), built from reference
    objects, B200 vs the oracle."""
    import copy
    pm = apps.gen_hex_mesh(94, seed=0)
    apps.shuffle_mesh(pm, seed=1)
    m = foreign.export_mesh(pm, R, auto_soa_threshold=thr)
    if renumber:
        R.renumber_mesh(m)
    mw = copy.deepcopy(m)
    prog, h = apps.build_hydra_proxy(m, steps=1, seed=0, api=R)
    progw, hw = apps.build_hydra_proxy(mw, steps=1, seed=0, api=R)
    assert {d.layout.name for d in m.dats.values() if d.dim > 1} == (
        {"AOS"} if thr is None else {"SOA"} if thr == 0 else {"AOS", "SOA"})
    b.run_program(prog, m, b.BackendConfig())
    bulk.run_program(progw)
    for k in ("q", "q_old", "res", "grad", "dt_loc"):
        _close(h[k].fetch(), hw[k].fetch(), k)
    assert h["dt_min"][0].value == hw["dt_min"][0].value
    _close(h["rms"][0].buffer, hw["rms"][0].buffer, "rms")


@pytest.mark.gpu
def test_reference_built_proxy_matches_stock_reference_small(R):
    """The proxy program built from reference objects: B200 vs the stock
    reference's own serial executor (per-element Python kernels)."""
    pm = apps.gen_hex_mesh(12, seed=5)
    m, mw = foreign.export_mesh(pm, R), foreign.export_mesh(pm, R)
    prog, h = apps.build_hydra_proxy(m, steps=2, seed=5, api=R)
    progw, hw = apps.build_hydra_proxy(mw, steps=2, seed=5, api=R)
    foreign.install(R)
    R.run_program(prog, m, R.BackendConfig(backend="cuda"))
    R.run_program(progw, mw, R.BackendConfig())
    for k in ("q", "q_old", "res", "grad", "dt_loc"):
        _close(h[k].fetch(), hw[k].fetch(), k)
    for k in ("dt_min", "rms"):
        for g, w in zip(h[k], hw[k]):
            _close(g.buffer, w.buffer, k)
