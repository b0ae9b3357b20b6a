"""GPU parity: the B200 backend vs the reference golden vectors and the CPU oracle.

Bars: int64 results bit-exact; float64 outputs within
rtol=1e-12 (reference tests/test_acceptance.py:94-97) — for raw increment
accumulators, where colouring reorders cancelling sums, within
1e-12 * max|ref| of the same component as well (``close``).  Everything
runs through the public API ``run_program`` -> libmeshloop_b200.so.
"""
from __future__ import annotations

import numpy as np
import pytest

import _cases
import paper_1403_7209_b200 as ml
from conftest import golden
from oracle import bulk, serial as oserial
from paper_1403_7209_b200 import apps
from paper_1403_7209_b200.kernels import device_kernel

pytestmark = pytest.mark.gpu

RTOL = 1e-12


def close(got, ref, rtol=RTOL, what=""):
    """rtol 1e-12, plus an absolute floor of 1e-12 * max|ref| per component."""
    got, ref = np.asarray(got, dtype=np.float64), np.asarray(ref, dtype=np.float64)
    if ref.ndim == 2:
        floor = rtol * np.max(np.abs(ref), axis=0, initial=0.0)[None, :]
    else:
        floor = rtol * np.max(np.abs(ref), initial=0.0)
    bad = np.abs(got - ref) > rtol * np.abs(ref) + floor
    assert not bad.any(), f"{what}: {bad.sum()} mismatches, max |d| {np.max(np.abs(got - ref))}"


SCHEDULES = ("gather", "pfold", "colour")


def cfg(**kw):
    return ml.BackendConfig(**kw)


def _exec_cases():
    return [c for c in golden("exec.npz").index if c["app"] in ("diffusion", "cell-area")]


@pytest.mark.parametrize("case", _exec_cases(), ids=lambda c: c["name"])
@pytest.mark.parametrize("bs,sched", [(256, "pfold"), (16, "pfold"), (256, "gather"), (16, "gather"),
                                      (256, "colour"), (16, "colour")])
def test_apps_match_reference_golden(case, bs, sched):
    g = golden("exec.npz")
    mesh, prog, h = _cases.build_app(case["app"], case["n"], case["dtype"], case["steps"])
    res = ml.run_program(prog, mesh, cfg(block_size=bs, inc_schedule=sched))
    assert {r.loop for r in res.perf} == {l.name for l in prog}
    for k, v in _cases.app_results(case["app"], h).items():
        want = g[f"exec/{case['name']}/{k}"]
        if case["dtype"] == "int64":
            np.testing.assert_array_equal(v, want, k)
        else:
            close(v, want, what=k)


@pytest.mark.parametrize("bs", [1, 3, 32, 100, 256, 512, 1024])
def test_int64_diffusion_bit_exact_at_every_block_size(bs):
    g = golden("exec.npz")
    mesh, prog, h = _cases.build_app("diffusion", 8, "int64", 3)
    ml.run_program(prog, mesh, cfg(block_size=bs))
    np.testing.assert_array_equal(h["u"].fetch(), g["exec/diffusion_n8_int64_s3/u"])
    np.testing.assert_array_equal([r.value for r in h["residuals"]],
                                  g["exec/diffusion_n8_int64_s3/residuals"])


def test_renumbered_diffusion_matches_reference():
    g = golden("exec.npz")
    mesh = apps.gen_mesh(10)
    prog, h = apps.build_diffusion(mesh, 2, dtype="int64")
    ml.renumber_mesh(mesh)
    ml.run_program(prog, mesh, cfg())
    np.testing.assert_array_equal(h["u"].fetch(), g["exec/diffusion_renum_n10_int64/u"])


@pytest.mark.parametrize("soa", [4, None, 0])
def test_mixmax_soa_minmax_read_globals(soa):
    g = golden("exec.npz")
    mesh, loop, acc, lo, hi = _cases.mixmax_case(auto_soa_threshold=soa)
    ml.run_program([loop], mesh, cfg(block_size=8))
    np.testing.assert_array_equal(acc.fetch(), g["exec/mixmax/acc"])
    assert [lo.value, hi.value] == g["exec/mixmax/lohi"].tolist()


def test_fuzz_meshes_match_reference_and_oracle(rng):
    g = golden("exec.npz")
    for case in g.index:
        if case["app"] != "fuzz":
            continue
        mesh, loop = _cases.random_loop_mesh(np.random.default_rng(case["seed"]), max_elems=300)
        ml.run_program([loop], mesh, cfg(block_size=int(rng.choice([1, 7, 32, 256])),
                                         inc_schedule=str(rng.choice(SCHEDULES))))
        np.testing.assert_array_equal(mesh.dats["vals"].fetch(), g[f"exec/{case['name']}/vals"])
    for _ in range(20):
        seed = int(rng.integers(0, 2 ** 31))
        ref_mesh, ref_loop = _cases.random_loop_mesh(np.random.default_rng(seed), max_elems=5000)
        oserial.run_loop(ref_loop)
        mesh, loop = _cases.random_loop_mesh(np.random.default_rng(seed), max_elems=5000)
        ml.run_program([loop], mesh, cfg(block_size=int(rng.choice([1, 7, 64, 256, 1024])),
                                         inc_schedule=str(rng.choice(SCHEDULES))))
        np.testing.assert_array_equal(mesh.dats["vals"].fetch(), ref_mesh.dats["vals"].fetch())


@pytest.mark.parametrize("N,steps", [(5, 2), (7, 1)])
def test_proxy_matches_reference_golden(N, steps):
    g = golden("exec.npz")
    mesh = apps.gen_hex_mesh(N, seed=4)
    prog, h = apps.build_hydra_proxy(mesh, steps=steps, seed=4)
    ml.run_program(prog, mesh, cfg())
    name = f"proxy_hex{N}_s{steps}"
    for k in ("q", "q_old", "dt_loc"):
        close(h[k].fetch(), g[f"exec/{name}/{k}"], what=k)
    for k in ("res", "grad"):                # zeroed by the update loop: exact
        np.testing.assert_array_equal(h[k].fetch(), g[f"exec/{name}/{k}"])
    close([r.value for r in h["rms"]], g[f"exec/{name}/rms"], what="rms")
    np.testing.assert_array_equal([r.value for r in h["dt_min"]], g[f"exec/{name}/dt_min"])


def _proxy_pair(N, seed=0, renumber=True, shuffle=True, soa=4):
    out = []
    for _ in range(2):
        mesh = apps.gen_hex_mesh(N, seed=seed, auto_soa_threshold=soa)
        if shuffle:
            apps.shuffle_mesh(mesh, seed=seed + 1)
        prog, h = apps.build_hydra_proxy(mesh, steps=1, seed=seed)
        if renumber:
            ml.renumber_mesh(mesh)
        out.append((mesh, prog, h))
    return out


@pytest.mark.parametrize("soa", [4, None, 0])
@pytest.mark.parametrize("sched", ["gather", "pfold", "colour"])
def test_proxy_partial_iteration_raw_accumulators_vs_oracle(soa, sched):
    """Stop before the update so the raw INC accumulators (res, grad) are compared,
    for every layout (auto-SoA, all AoS, all SoA) and INC schedule."""
    (rm, rprog, rh), (mesh, prog, h) = _proxy_pair(16, soa=soa)
    bulk.run_program(rprog[:5])
    ml.run_program(prog[:5], mesh, cfg(inc_schedule=sched))
    for k in ("grad", "res", "q_old", "dt_loc"):
        close(h[k].fetch(), rh[k].fetch(), what=k)
    np.testing.assert_array_equal(h["dt_min"][0].value, rh["dt_min"][0].value)


@pytest.mark.parametrize("sched", ["pfold", "gather", "colour"])
def test_proxy_full_size_iteration_vs_oracle(sched):
    """Config B (Rotor37-sized, 2.47M edges): one full iteration, shuffled + CM-renumbered."""
    (rm, rprog, rh), (mesh, prog, h) = _proxy_pair(94, seed=0)
    bulk.run_program(rprog)
    ml.run_program(prog, mesh, cfg(inc_schedule=sched))
    close(h["q"].fetch(), rh["q"].fetch(), what="q")
    close([h["rms"][0].value], [rh["rms"][0].value], what="rms")
    assert h["dt_min"][0].value == rh["dt_min"][0].value


def test_int64_diffusion_rotor37_size_bit_exact():
    """gen_mesh(913): 835,396 nodes / 2,502,533 edges, int64 twin, bit-exact vs oracle."""
    ref = apps.gen_mesh(913)
    rprog, rh = apps.build_diffusion(ref, 2, dtype="int64")
    bulk.run_program(rprog)
    mesh = apps.gen_mesh(913)
    prog, h = apps.build_diffusion(mesh, 2, dtype="int64")
    ml.run_program(prog, mesh, cfg())
    np.testing.assert_array_equal(h["u"].fetch(), rh["u"].fetch())
    assert [r.value for r in h["residuals"]] == [r.value for r in rh["residuals"]]


def test_colouring_stress_hub_and_shuffled_meshes():
    for make in (lambda: apps.gen_hub_mesh(20000, 200000, n_hubs=4, hub_share=0.05, seed=2),
                 lambda: _shuffled_hex(30)):
        ref, mesh = make(), make()
        rl = _cases.inc_loop(ref, "edge_nodes")
        oserial.run_loop(rl)
        want = ref.dats["acc"].fetch()
        for sched in SCHEDULES:
            l = _cases.inc_loop(mesh, "edge_nodes")
            mesh.dats["acc"].put(np.zeros_like(want))
            res = ml.run_program([l], mesh, cfg(inc_schedule=sched))
            np.testing.assert_array_equal(mesh.dats["acc"].fetch(), want, sched)
        assert res.perf[0].nc > 8


def _shuffled_hex(N):
    m = apps.gen_hex_mesh(N)
    apps.shuffle_mesh(m, seed=9)
    return m


def test_empty_iteration_set_is_a_noop():
    mesh = ml.Mesh()
    nodes = mesh.decl_set("nodes", 5)
    none = mesh.decl_set("none", 0)
    m = mesh.decl_map("en", none, nodes, 1, [])
    vals = mesh.decl_dat("vals", nodes, 1, "int64", np.arange(5))
    loop = _cases.inc_loop(mesh, "en", "vals")
    total = ml.Global(np.int64(7))
    z = mesh.decl_dat("z", none, 1, "int64", [])
    cnt = ml.Loop("cnt", none, [ml.arg_direct(z, ml.READ), ml.arg_global(total, ml.INC)],
                  apps._k_sum)
    ml.run_program([loop, cnt], mesh, cfg())
    np.testing.assert_array_equal(vals.fetch().ravel(), np.arange(5))
    assert total.value == 7


def test_direct_loop_is_exact_even_in_float():
    @device_kernel("scale_rw")
    def scale(v):
        v[0] = v[0] * 1.0000001 + 0.25
    mesh = ml.Mesh()
    d = mesh.decl_dat("d", mesh.decl_set("s", 100000), 1, "float64", np.linspace(0.0, 1.0, 100000))
    want = np.linspace(0.0, 1.0, 100000) * 1.0000001 + 0.25
    ml.run_program([ml.Loop("scale", d.set, [ml.arg_direct(d, ml.RW)], scale)], mesh, cfg(block_size=64))
    np.testing.assert_array_equal(d.fetch().ravel(), want)


def test_float_results_are_deterministic_run_to_run():
    outs = []
    for _ in range(2):
        mesh = apps.gen_hex_mesh(24, seed=1)
        prog, h = apps.build_hydra_proxy(mesh, steps=3, seed=1)
        ml.run_program(prog, mesh, cfg())
        outs.append((h["q"].fetch(), [r.value for r in h["rms"]]))
    np.testing.assert_array_equal(outs[0][0], outs[1][0])
    assert outs[0][1] == outs[1][1]


def test_graph_replay_and_host_residency_match_eager():
    results = []
    for kw in ({}, {"use_graph": True}, {"residency": "host"},
               {"residency": "host", "use_graph": True}, {"residency": "host", "time_loops": False}):
        mesh = apps.gen_hex_mesh(12, seed=2)
        prog, h = apps.build_hydra_proxy(mesh, steps=1, seed=2)
        for _ in range(3):                   # replayed: state advances identically
            ml.run_program(prog, mesh, cfg(**kw))
            if kw.get("residency") == "host":     # host edits between runs are uploaded
                assert not h["q"]._dev.device_newer
        results.append((h["q"].fetch(), h["rms"][0].value, h["res"].fetch(), h["q_old"].fetch()))
    for q, r, res, qo in results[1:]:
        np.testing.assert_array_equal(q, results[0][0])
        assert r == results[0][1]
        np.testing.assert_array_equal(res, results[0][2])
        np.testing.assert_array_equal(qo, results[0][3])


@pytest.mark.parametrize("soa,sched", [(4, "gather"), (None, "gather"), (0, "gather")])
def test_gather_schedule_reproduces_serial_order_bitwise(soa, sched):
    """Target-centric schedule accumulates every target in the reference serial
    order, so even float64 raw INC accumulators equal the oracle bit for bit."""
    (rm, rprog, rh), (mesh, prog, h) = _proxy_pair(20, soa=soa)
    bulk.run_program(rprog[:5])
    # unchained: a chained iflux+vflux interleaves the two loops' increments
    ml.run_program(prog[:5], mesh, cfg(inc_schedule=sched, chain_loops=False))
    for k in ("grad", "res", "q_old", "dt_loc"):
        np.testing.assert_array_equal(h[k].fetch(), rh[k].fetch(), k)
    (rm, rprog, rh), (mesh, prog, h) = _proxy_pair(16, seed=3)
    bulk.run_program(rprog)
    ml.run_program(prog, mesh, cfg(inc_schedule=sched))
    close(h["q"].fetch(), rh["q"].fetch(), what="q")
    for app in ("diffusion", "cell-area"):
        g = golden("exec.npz")
        mesh, p, hh = _cases.build_app(app, 8 if app == "diffusion" else 6, "float64",
                                       3 if app == "diffusion" else 0)
        ml.run_program(p, mesh, cfg(inc_schedule=sched))
        name = f"{app}_n{8 if app == 'diffusion' else 6}_float64_s{3 if app == 'diffusion' else 0}"
        for k, v in _cases.app_results(app, hh).items():
            close(v, g[f"exec/{name}/{k}"], what=k)
    for make in (lambda: apps.gen_hub_mesh(5000, 60000, n_hubs=8, hub_share=0.2, seed=3),
                 lambda: _shuffled_hex(16)):
        ref, mesh = make(), make()
        oserial.run_loop(_cases.inc_loop(ref, "edge_nodes"))
        ml.run_program([_cases.inc_loop(mesh, "edge_nodes")], mesh, cfg(inc_schedule=sched))
        np.testing.assert_array_equal(mesh.dats["acc"].fetch(), ref.dats["acc"].fetch())
    mesh, loop, acc, lo, hi = _cases.mixmax_case()
    ml.run_program([loop], mesh, cfg(inc_schedule=sched))
    gg = golden("exec.npz")
    np.testing.assert_array_equal(acc.fetch(), gg["exec/mixmax/acc"])
    assert [lo.value, hi.value] == gg["exec/mixmax/lohi"].tolist()


def test_host_writes_between_runs_are_uploaded():
    mesh = apps.gen_mesh(6)
    prog, h = apps.build_diffusion(mesh, 1, dtype="int64")
    ml.run_program(prog, mesh, cfg())
    h["u"].put(np.zeros((mesh.sets["nodes"].size, 1), np.int64))      # host write
    h["bc_values"].data[:] = 0                                        # write through .data
    h["residuals"][0].buffer[:] = 0
    ml.run_program(prog, mesh, cfg())
    assert h["residuals"][0].value == 0
    np.testing.assert_array_equal(h["u"].fetch(), 0)


def test_unbound_kernel_raises_exec_error():
    mesh = ml.Mesh()
    d = mesh.decl_dat("d", mesh.decl_set("s", 4), 1, "float64", np.zeros(4))
    with pytest.raises(ml.ExecError, match="no device functor"):
        ml.run_program([ml.Loop("x", d.set, [ml.arg_direct(d, ml.RW)], lambda v: None)], mesh)


def test_signature_mismatch_raises_exec_error():
    mesh = ml.Mesh()
    s = mesh.decl_set("s", 4)
    d = mesh.decl_dat("d", s, 2, "float64", np.zeros(8))
    with pytest.raises(ml.ExecError, match="takes 2 args"):
        ml.run_program([ml.Loop("x", s, [ml.arg_direct(d, ml.RW)], apps._k_copy)], mesh)


def test_perf_records_and_report_schema(tmp_path):
    import json
    mesh = apps.gen_mesh(16)
    prog, _ = apps.build_cell_area(mesh, "float64")
    out = ml.run_program(prog, mesh, cfg())
    assert sum(r.pct_runtime for r in out.perf) == pytest.approx(100.0, abs=0.01)
    assert all(r.time_sec > 0 and r.gb_per_sec > 0 for r in out.perf)
    path = tmp_path / "r.json"
    ml.emit_report(out.perf, path, config={"backend": "cuda"},
                   mesh_sets={n: s.size for n, s in mesh.sets.items()})
    assert {l["loop"] for l in json.loads(path.read_text())["loops"]} == \
        {"area_calc", "area_distribute", "area_total"}


def test_reference_per_loop_entries():
    """run_serial reproduces the serial order bit for bit (gather schedule);
    run_threads is the coloured schedule; run_hybrid refuses loudly."""
    ref, a, b = apps.gen_hub_mesh(3000, 30000, n_hubs=4, hub_share=0.1, seed=5), None, None
    ref.decl_dat("acc", ref.sets["nodes"], 1, "float64", np.zeros(ref.sets["nodes"].size))
    a = apps.gen_hub_mesh(3000, 30000, n_hubs=4, hub_share=0.1, seed=5)
    a.decl_dat("acc", a.sets["nodes"], 1, "float64", np.zeros(a.sets["nodes"].size))
    b = apps.gen_hub_mesh(3000, 30000, n_hubs=4, hub_share=0.1, seed=5)
    b.decl_dat("acc", b.sets["nodes"], 1, "float64", np.zeros(b.sets["nodes"].size))
    oserial.run_loop(_cases.inc_loop(ref, "edge_nodes", dtype="float64"))
    ml.run_serial(_cases.inc_loop(a, "edge_nodes", dtype="float64"), a)
    np.testing.assert_array_equal(a.dats["acc"].fetch(), ref.dats["acc"].fetch())
    ml.run_threads(_cases.inc_loop(b, "edge_nodes", dtype="float64"), b)
    close(b.dats["acc"].fetch(), ref.dats["acc"].fetch(), what="threads")
    with pytest.raises(ml.ExecError, match="run_hybrid"):
        ml.run_hybrid([], b)


@pytest.mark.parametrize("seed", [0, 1, 2, 3])
def test_gather_write_is_serial_last_writer(seed):
    """Indirect WRITE loops with conflicting writers: the gather schedule keeps the
    serial order's last writer per target (compacted target list when sparse)."""
    rng = np.random.default_rng(seed)
    for max_elems in (50, 5000, 40000):
        ref, _ = _cases.random_loop_mesh(np.random.default_rng(seed * 7 + max_elems), max_elems)
        mesh, _ = _cases.random_loop_mesh(np.random.default_rng(seed * 7 + max_elems), max_elems)
        oserial.run_loop(_cases.write_loop(ref))
        ml.run_program([_cases.write_loop(mesh)], mesh,
                       cfg(block_size=int(rng.choice([7, 64, 256]))))
        np.testing.assert_array_equal(mesh.dats["vals"].fetch(), ref.dats["vals"].fetch())


def test_pfold_schedule_raw_accumulators_reductions_and_determinism():
    """Primary fold: raw INC accumulators within tolerance of the serial oracle,
    int64 bit-exact (fuzz + diffusion), MIN/MAX/READ globals counted once per
    element, bitwise run to run."""
    (rm, rprog, rh), (mesh, prog, h) = _proxy_pair(12)
    bulk.run_program(rprog[:5])
    c = cfg(inc_schedule="pfold")
    ml.run_program(prog[:5], mesh, c)
    for k in ("grad", "res"):
        close(h[k].fetch(), rh[k].fetch(), what=k)
    first = {k: h[k].fetch().copy() for k in ("grad", "res")}
    for k in ("grad", "res"):
        h[k].data[...] = 0.0
    ml.run_program(prog[:5], mesh, c)
    for k in ("grad", "res"):
        np.testing.assert_array_equal(h[k].fetch(), first[k])
    g = golden("exec.npz")
    for soa in (4, None):
        mesh, loop, acc, lo, hi = _cases.mixmax_case(auto_soa_threshold=soa)
        ml.run_program([loop], mesh, cfg(inc_schedule="pfold"))
        np.testing.assert_array_equal(acc.fetch(), g["exec/mixmax/acc"])
        assert [lo.value, hi.value] == g["exec/mixmax/lohi"].tolist()
    rng = np.random.default_rng(11)
    for _ in range(10):
        seed = int(rng.integers(0, 2 ** 31))
        ref_mesh, ref_loop = _cases.random_loop_mesh(np.random.default_rng(seed), max_elems=3000)
        oserial.run_loop(ref_loop)
        mesh, loop = _cases.random_loop_mesh(np.random.default_rng(seed), max_elems=3000)
        ml.run_program([loop], mesh, cfg(inc_schedule="pfold"))
        np.testing.assert_array_equal(mesh.dats["vals"].fetch(), ref_mesh.dats["vals"].fetch())


def test_concurrent_loops_match_sequential_and_respect_the_dag():
    """Independent loops overlap on streams (graphs / untimed runs); every dat and
    global sees the same sequence of writers, so results are bitwise the
    sequential ones.  The DAG: iflux does not wait for grad_edge (disjoint
    writes, no shared written buffer); vflux waits for both (reads grad, INCs res)."""
    from paper_1403_7209_b200.executor import compile_program
    for chain in (False, True):
        results = []
        for conc, graph in ((False, True), (True, True), (True, False), (False, False)):
            mesh = apps.gen_hex_mesh(16, seed=2)
            prog, h = apps.build_hydra_proxy(mesh, steps=2, seed=2)
            for _ in range(2):
                ml.run_program(prog, mesh, cfg(use_graph=graph, time_loops=False, concurrent_loops=conc,
                                               chain_loops=chain))
            results.append((h["q"].fetch(), [g.value for g in h["rms"]], [g.value for g in h["dt_min"]]))
        for q, rms, dt in results[1:]:
            np.testing.assert_array_equal(q, results[0][0])
            assert rms == results[0][1] and dt == results[0][2]
    cp = compile_program(prog, mesh, cfg(use_graph=True, chain_loops=False))
    names = [e.loop.name for e in cp.entries]
    deps = cp.dependencies()
    g, i, v = names.index("grad_edge"), names.index("iflux"), names.index("vflux")
    assert g not in deps[i][0]
    assert g in deps[v][0] and i in deps[v][0]
    assert deps[i][1] != deps[g][1]                      # they run on different streams


@pytest.mark.parametrize("sched", ["gather", "pfold", "colour"])
def test_chained_flux_loops_match_oracle(sched):
    """iflux+vflux chained into one loop (chain.py): raw res accumulators within
    the reference tolerance of the serial oracle running the loops one by one,
    the same as the unchained run within tolerance, bitwise run to run; the
    full iteration's q, rms and dt_min too."""
    from paper_1403_7209_b200.executor import compile_program
    (rm, rprog, rh), (mesh, prog, h) = _proxy_pair(16, seed=5)
    bulk.run_program(rprog[:5])
    c = cfg(inc_schedule=sched)
    assert [l.name for l in compile_program(prog[:5], mesh, c).run_loops][-1] == "iflux+vflux"
    ml.run_program(prog[:5], mesh, c)
    for k in ("grad", "res", "q_old", "dt_loc"):
        close(h[k].fetch(), rh[k].fetch(), what=k)
    first = h["res"].fetch().copy()
    h["res"].data[...] = 0.0
    (m2, p2, h2), _ = _proxy_pair(16, seed=5)
    ml.run_program(p2[:5], m2, cfg(inc_schedule=sched, chain_loops=False))
    close(first, h2["res"].fetch(), what="res chained vs unchained")
    ml.run_program(prog[3:5], mesh, c)
    np.testing.assert_array_equal(h["res"].fetch(), first)
    (rm, rprog, rh), (mesh, prog, h) = _proxy_pair(16, seed=6)
    bulk.run_program(rprog)
    ml.run_program(prog, mesh, cfg(inc_schedule=sched, use_graph=True))
    close(h["q"].fetch(), rh["q"].fetch(), what="q")
    close([h["rms"][0].value], [rh["rms"][0].value], what="rms")
    assert h["dt_min"][0].value == rh["dt_min"][0].value


@pytest.mark.parametrize("sched", ["auto", "pfold"])
def test_config_d_8m_edges_int64_bit_exact(sched):
    """Config D (gen_mesh(1633): 2,669,956 nodes / 8,003,333 edges), int64
    diffusion twin, two steps: bit-exact vs the oracle at the largest
    single-GPU size BASELINE.json names."""
    ref = apps.gen_mesh(1633)
    rprog, rh = apps.build_diffusion(ref, 2, dtype="int64")
    bulk.run_program(rprog)
    mesh = apps.gen_mesh(1633)
    prog, h = apps.build_diffusion(mesh, 2, dtype="int64")
    ml.run_program(prog, mesh, cfg(inc_schedule=sched))
    np.testing.assert_array_equal(h["u"].fetch(), rh["u"].fetch())
    assert [r.value for r in h["residuals"]] == [r.value for r in rh["residuals"]]


def test_config_d_proxy_iteration_vs_oracle():
    """139^3 grid (7,998,894 edges): one chained Hydra-proxy iteration with the
    default schedules vs the oracle running the loops one by one."""
    (rm, rprog, rh), (mesh, prog, h) = _proxy_pair(139, seed=2)
    bulk.run_program(rprog)
    ml.run_program(prog, mesh, cfg())
    close(h["q"].fetch(), rh["q"].fetch(), what="q")
    close([h["rms"][0].value], [rh["rms"][0].value], what="rms")
    assert h["dt_min"][0].value == rh["dt_min"][0].value




def test_phase_callback_instruments_each_colour_phase():
    """Reference tests/test_executor.py:324-364 instruments the threads
    backend's colour phases with BackendConfig.phase_callback.  Here the
    callback fires before each block colour's launch (colour schedule) and the
    device state between two callbacks shows exactly the increments of that
    colour's blocks; the result equals the serial oracle."""
    import ctypes as C
    from paper_1403_7209_b200 import _native as N
    from paper_1403_7209_b200.plan import plan_for
    ref = apps.gen_mesh(12)
    oserial.run_loop(_cases.inc_loop(ref, "edge_nodes"))
    mesh = apps.gen_mesh(12)
    loop = _cases.inc_loop(mesh, "edge_nodes")
    acc = mesh.dats["acc"]
    bs = 16
    snaps, calls = [], []

    def device_acc():
        m = acc._dev
        out = np.empty(acc.set.size, np.int64)
        N.check(N.lib().ml_download(N.ptr(out), m.ptr, out.nbytes))
        return out

    def cb(name, colour):
        calls.append((name, colour))
        snaps.append(device_acc())

    ml.run_threads(loop, mesh, cfg(block_size=bs, phase_callback=cb))
    plan = plan_for(loop, mesh, bs)
    assert calls == [(loop.name, c) for c in range(plan.ncolors)] and plan.ncolors > 1
    snaps.append(acc.fetch().ravel())
    np.testing.assert_array_equal(snaps[-1], ref.dats["acc"].fetch().ravel())
    table = mesh.maps["edge_nodes"].table
    for c in range(plan.ncolors):
        blocks = np.flatnonzero(plan.block_color == c)
        elems = np.concatenate([np.arange(b * bs, min((b + 1) * bs, table.shape[0])) for b in blocks])
        touched = np.unique(table[elems].ravel())
        changed = np.flatnonzero(snaps[c + 1] != snaps[c])
        assert set(changed) <= set(touched)
    # loops on the target-centric schedules have no colour phases
    calls.clear()
    ml.run_program([_cases.inc_loop(mesh, "edge_nodes")], mesh, cfg(phase_callback=cb, inc_schedule="gather"))
    assert calls == []
