"""Host-side product logic vs the reference golden vectors and the oracle (CPU).

Covers the C++ plan builder (ml_plan_build), the C++ Cuthill–McKee
renumbering (ml_co_occurrence / ml_cm_order), the vectorised partition and
halo builders, and the byte model — all bit-exact integer work."""
from __future__ import annotations

import numpy as np
import pytest

import _cases
import paper_1403_7209_b200 as ml
from conftest import golden, golden_bytes
from oracle import plan as oplan
from paper_1403_7209_b200 import apps
from paper_1403_7209_b200.executor import BackendConfig
from paper_1403_7209_b200.partition import derive_assignments


def test_native_plan_matches_reference_golden():
    g = golden("plans.npz")
    for case in g.index:
        name = case["name"]
        cols = [(k, g[f"plan/{name}/col{j}"]) for j, k in enumerate(case["keys"])]
        p = ml.build_plan(case["n"], cols, case["bs"])
        np.testing.assert_array_equal(p.block_color, g[f"plan/{name}/block_color"], name)
        np.testing.assert_array_equal(p.elem_color, g[f"plan/{name}/elem_color"], name)
        np.testing.assert_array_equal(p.elem_ncolors, g[f"plan/{name}/elem_ncolors"], name)
        assert p.ncolors == int(g[f"plan/{name}/ncolors"]), name
        np.testing.assert_array_equal(p.blocks_flat, g[f"plan/{name}/blocks_by_color"], name)
        np.testing.assert_array_equal(np.diff(p.color_offsets), g[f"plan/{name}/bpc"], name)
        np.testing.assert_array_equal(p.elem_order_flat, g[f"plan/{name}/block_elem_order"], name)
        flat = np.concatenate(p.block_elem_order) if p.nblocks else np.zeros(0, np.int64)
        np.testing.assert_array_equal(flat, g[f"plan/{name}/block_elem_order"], name)


def test_native_plan_matches_oracle_on_fuzz(rng):
    for _ in range(25):
        mesh, loop = _cases.random_loop_mesh(rng, max_elems=600)
        bs = int(rng.choice([1, 2, 7, 16, 64, 256]))
        cols = oplan.write_columns(loop)
        got = ml.build_plan(loop.iter_set.size, cols, bs)
        want = oplan.build_plan(loop.iter_set.size, cols, bs)
        np.testing.assert_array_equal(got.block_color, want.block_color)
        np.testing.assert_array_equal(got.elem_color, want.elem_color)
        np.testing.assert_array_equal(got.elem_ncolors, want.elem_ncolors)


def test_native_plan_is_race_free_exhaustive(rng):
    """Independent conflict scan (reference tests/conftest.py:137-160)."""
    for _ in range(20):
        mesh, loop = _cases.random_loop_mesh(rng, max_elems=300)
        bs = int(rng.choice([1, 3, 16, 64]))
        p = ml.plan_for(loop, mesh, bs)
        targets = lambda e: {(a.dat.name, int(a.map.table[e, a.slot])) for a in loop.args
                             if a.kind == "indirect" and a.writes}
        assert oplan.race_free(p, targets)


def test_plan_cache_counts_builds_and_reuses():
    mesh = apps.sample_mesh()
    loop = _cases.inc_loop(mesh, "cell_nodes")
    assert mesh._plan_builds == 0
    p1 = ml.plan_for(loop, mesh, 4)
    assert ml.plan_for(loop, mesh, 4) is p1 and mesh._plan_builds == 1
    ml.plan_for(loop, mesh, 8)
    assert mesh._plan_builds == 2
    assert ml.plan_for(_cases.inc_loop(mesh, "cell_nodes"), mesh, 4) is p1


def test_plan_known_answers():
    mesh = ml.Mesh()
    nodes = mesh.decl_set("nodes", 1)
    edges = mesh.decl_set("edges", 3)
    mesh.decl_map("en", edges, nodes, 1, [1, 1, 1])
    loop = _cases.inc_loop(mesh, "en")
    st = ml.plan_stats(ml.plan_for(loop, mesh, 1))
    assert (st.nb, st.nc, st.blocks_per_color) == (3, 3, [1, 1, 1])
    p = ml.plan_for(loop, mesh, 8)
    assert p.nblocks == 1 and p.ncolors == 1 and p.elem_ncolors[0] == 3
    sm = apps.sample_mesh()
    p = ml.plan_for(_cases.inc_loop(sm, "cell_nodes"), sm, 4)
    assert p.block_bounds.tolist() == [0, 4, 8, 12, 16, 17]
    with pytest.raises(ValueError):
        ml.build_plan(4, [], 0)


def test_block_count_halves_colours_banded_gen64():
    """reference acceptance criterion 9 (tests/test_acceptance.py:269-282)."""
    mesh = apps.gen_mesh(64)
    prog, _ = apps.build_diffusion(mesh, 1, dtype="int64")
    flux = next(l for l in prog if l.name == "edge_flux")
    prev = None
    for bs in (64, 128, 256, 512, 1024, 2048):
        st = ml.plan_stats(ml.plan_for(flux, mesh, bs))
        if prev is not None:
            assert abs(prev / 2 - st.nb) <= 1
        assert 4 <= st.nc <= 24
        prev = st.nb


# -- renumbering ---------------------------------------------------------------------

def _product_mesh_from_golden(g, case):
    name = case["name"]
    mesh = ml.Mesh()
    sets = {n: mesh.decl_set(n, s) for n, s in case["sets"].items()}
    for mn, f, t, a in case["maps"]:
        mesh.decl_map(mn, sets[f], sets[t], a, (g[f"ren/{name}/table/{mn}"] + 1).ravel())
    return mesh


def test_native_cm_ordering_matches_reference_golden():
    g = golden("renumber.npz")
    for case in g.index:
        if f"ren/{case['name']}/cm_forward" not in g:
            continue
        mesh = _product_mesh_from_golden(g, case)
        perm = ml.compute_ordering(mesh, mesh.sets["nodes"])
        np.testing.assert_array_equal(perm.forward, g[f"ren/{case['name']}/cm_forward"])


def test_native_renumber_mesh_matches_reference_golden():
    g = golden("renumber.npz")
    for case in g.index:
        mesh = _product_mesh_from_golden(g, case)
        rep = ml.renumber_mesh(mesh)
        assert sorted(rep["permutations"]) == sorted(case["perm_sets"])
        for s, p in rep["permutations"].items():
            np.testing.assert_array_equal(p.forward, g[f"ren/{case['name']}/full/{s}"], s)
        for mn, (b, a) in rep["maps"].items():
            key = f"ren/{case['name']}/span/{mn}"
            if key in g:
                np.testing.assert_allclose([b.max_span, b.mean_span, a.max_span, a.mean_span], g[key])


def test_renumber_api_contract():
    mesh = _cases.path_mesh()
    assert ml.compute_ordering(mesh, mesh.sets["nodes"]).is_identity()
    mesh = _cases.path_mesh((3, 1, 4, 2))
    ml.apply_permutation(mesh, ml.compute_ordering(mesh, mesh.sets["nodes"]))
    assert ml.bandwidth_metric(mesh, mesh.maps["edge_nodes"]).max_span == 1
    sm = apps.sample_mesh()
    perm = ml.compute_ordering(sm, sm.sets["nodes"])
    sm.decl_set("other", 3)
    with pytest.raises(ml.MeshError, match="stale"):
        ml.apply_permutation(sm, perm)
    lonely = ml.Mesh()
    s = lonely.decl_set("lonely", 5)
    with pytest.raises(ml.MeshError, match="no incident map"):
        ml.compute_ordering(lonely, s)
    sm = apps.sample_mesh()
    f = np.arange(14)
    f[0], f[1] = 1, 0
    ml.apply_permutation(sm, ml.Permutation("nodes", f, f.copy(), sm.version))
    assert (sm.maps["cell_nodes"].table[:2] + 1).ravel().tolist() == [2, 3, 10, 2, 1, 3]
    m = ml.Mesh()
    nodes = m.decl_set("nodes", 5)
    edges = m.decl_set("edges", 4)
    en = m.decl_map("en", edges, nodes, 2, [3, 4, 1, 2, 3, 1, 1, 2])
    ml.apply_permutation(m, ml.row_order_by_targets(m, en))
    assert (m.maps["en"].table + 1).tolist() == [[1, 2], [1, 2], [3, 1], [3, 4]]


def test_renumbering_cuts_span_on_shuffled_mesh():
    """reference acceptance criterion 4 (span cut >= 30 %)."""
    mesh = apps.gen_mesh(64)
    apps.shuffle_mesh(mesh, seed=4, sets=["nodes", "edges"])
    shuffled = ml.bandwidth_metric(mesh, mesh.maps["edge_nodes"])
    rep = ml.renumber_mesh(mesh)
    assert 1.0 - rep["maps"]["edge_nodes"][1].mean_span / shuffled.mean_span >= 0.30


# -- partitions / halos ------------------------------------------------------------------

def test_partitioners_match_reference_golden():
    g = golden("partition.npz")
    for name in ("rand64_2d", "rand50_2d_tie", "rand200_3d"):
        xy = g[f"part/{name}/xy"]
        m = ml.Mesh()
        s = m.decl_set("pts", xy.shape[0])
        c = m.decl_dat("coords", s, xy.shape[1], "float64", xy.ravel())
        for nr in (2, 4, 8):
            np.testing.assert_array_equal(ml.partition_rcb(c, nr).rank_of, g[f"part/{name}/rcb{nr}"])
    for size, nr in ((17, 2), (14, 1), (4, 8), (1001, 8)):
        got = ml.partition_trivial(ml.Mesh().decl_set("s", size), nr).rank_of
        np.testing.assert_array_equal(got, g[f"part/trivial_{size}_{nr}"])
    with pytest.raises(ml.MeshError, match="power-of-two"):
        ml.partition_rcb(c, 3)
    assert ml.partition_weighted(ml.Mesh().decl_set("s", 7000), [5.0, 1.0, 1.0]).sizes() == \
        [5000, 1000, 1000]


def _layout_for(case):
    mesh, prog, _ = _cases.build_app(case["app"], case["n"], "int64", 1)
    nr = case["nranks"]
    targets = []
    for l in prog:
        for a in l.args:
            if a.kind == "indirect" and a.map.to_set not in targets:
                targets.append(a.map.to_set)
    base = {}
    for t in targets:
        base[t.name] = (ml.partition_rcb(mesh.dats["coords"], nr) if case["partitioner"] == "rcb"
                        else ml.partition_trivial(t, nr))
    seen, loops = set(), []
    for l in prog:
        if l.signature() not in seen:
            seen.add(l.signature())
            loops.append(l)
    return ml.build_halos(mesh, loops, derive_assignments(mesh, loops, base, nr))


def _assert_layout(g, key, lay):
    for sname, per in lay.sets.items():
        for r, h in enumerate(per):
            for part, arr in (("owned", h.owned), ("exec", h.exec_halo), ("nonexec", h.nonexec_halo)):
                np.testing.assert_array_equal(arr, g[f"{key}/{sname}/{r}/{part}"], f"{key} {sname} {r}")
            assert sorted(h.imports) == sorted(int(k.rsplit("imp", 1)[1])
                                               for k in g.keys(f"{key}/{sname}/{r}/imp"))
            for q, ids in h.imports.items():
                np.testing.assert_array_equal(ids, g[f"{key}/{sname}/{r}/imp{q}"])
            for q, ids in h.exports.items():
                np.testing.assert_array_equal(ids, g[f"{key}/{sname}/{r}/exp{q}"])


def test_layouts_match_reference_golden():
    g = golden("partition.npz")
    for case in g.index:
        if case["app"] == "fuzz":
            nt, ni = case["sizes"]
            table = g[f"fuzzlay/{case['name'][4:]}/table"]
            mesh = ml.Mesh()
            tgt, it = mesh.decl_set("tgt", nt), mesh.decl_set("it", ni)
            m = mesh.decl_map("m", it, tgt, table.shape[1], (table + 1).ravel())
            vals = mesh.decl_dat("vals", tgt, 1, "int64", np.zeros(nt, np.int64))
            src = mesh.decl_dat("src", it, 1, "int64", np.zeros(ni, np.int64))
            loop = ml.Loop("fuzz", it, [ml.arg_direct(src, ml.READ)] +
                           [ml.arg_indirect(vals, m, k + 1, ml.INC) for k in range(table.shape[1])],
                           lambda *a: None)
            nr = case["nranks"]
            asg = derive_assignments(mesh, [loop], {"tgt": ml.partition_trivial(tgt, nr)}, nr)
            lay = ml.build_halos(mesh, [loop], asg)
        else:
            lay = _layout_for(case)
        _assert_layout(g, f"lay/{case['name']}", lay)


def test_halo_mirror_symmetry_and_unassigned_error(rng):
    mesh, loop = _cases.random_loop_mesh(rng, max_elems=200)
    asg = derive_assignments(mesh, [loop], {"tgt": ml.partition_trivial(mesh.sets["tgt"], 4)}, 4)
    lay = ml.build_halos(mesh, [loop], asg)
    for per in lay.sets.values():
        for r, h in enumerate(per):
            for src, ids in h.imports.items():
                np.testing.assert_array_equal(ids, per[src].exports[r])
    pm = _cases.path_mesh()
    with pytest.raises(ml.MeshError, match="unassigned"):
        ml.build_halos(pm, [_cases.inc_loop(pm)], {"edges": ml.partition_trivial(pm.sets["edges"], 2)})


# -- bytes ----------------------------------------------------------------------------------

def test_useful_bytes_match_reference():
    want = golden_bytes()
    m = apps.gen_hex_mesh(12, seed=1)
    prog, _ = apps.build_hydra_proxy(m, steps=1)
    assert {l.name: ml.useful_bytes(l) for l in prog} == want["hex12_proxy"]
    m = apps.gen_mesh(64)
    prog, _ = apps.build_diffusion(m, 1)
    assert {l.name: ml.useful_bytes(l) for l in prog} == want["gen64_diffusion"]
    flux = next(l for l in prog if l.name == "edge_flux")
    assert ml.b_alg(flux) == want["gen64_diffusion"]["edge_flux"] + 4 * 2 * flux.iter_set.size


def test_backend_config_validation():
    with pytest.raises(ml.MeshError, match="unknown backend"):
        BackendConfig(backend="threads")
    with pytest.raises(ml.MeshError):
        BackendConfig(block_size=0)
    with pytest.raises(ml.MeshError, match="partitioner"):
        BackendConfig(partitioner="metis")
    assert BackendConfig(block_size_table={"a": 64}).block_size_for("a") == 64


def test_gather_hub_rows_and_pfold_lists(rng):
    """Gather lists with hub splitting: every target's incidences covered once,
    in serial order, rows of <= hub_row; pfold lists = the position-0 / >0
    incidences per target, element ascending."""
    from paper_1403_7209_b200.device import gather_lists_host, pfold_lists_host
    for trial in range(6):
        mesh = apps.gen_hub_mesh(300, 4000, n_hubs=3, hub_share=0.3, seed=trial)
        prog, _ = apps.build_diffusion(mesh, 1, dtype="int64")
        loop = prog[1]
        n = loop.iter_set.size
        tab = mesh.maps["edge_nodes"].table
        for hub_row in (7, 128):
            h = gather_lists_host(loop, n, hubs=True, hub_row=hub_row)
            off, elem, pos = h["off"], h["elem"], h["pos"]
            tl = h["targets"] if h["targets"] is not None else np.arange(off.size - 1)
            assert np.all(np.diff(off) <= hub_row) or h["seg"] is None
            got = {}
            for r in range(off.size - 1):
                got.setdefault(int(tl[r]), []).extend(
                    zip(elem[off[r]:off[r + 1]].tolist(), pos[off[r]:off[r + 1]].tolist()))
            want = {}
            for e in range(n):
                for a in range(2):
                    want.setdefault(int(tab[e, a]), []).append((e, a))
            assert got == want
            if h["seg"] is not None:
                seg = h["seg"]
                assert sorted(seg[seg >= 0].tolist()) == list(range(h["nslots"]))
                for k, t in enumerate(h["hub_tl"]):
                    rows = np.flatnonzero((tl == t) & (seg >= 0))
                    assert seg[rows].tolist() == list(range(h["hub_off"][k], h["hub_off"][k + 1]))
            pf = pfold_lists_host(h["host"], hub_row=None)
            # primary incidence = the element's first INC argument
            prim_pos = np.zeros(n, np.int64)
            k = np.arange(pf["elem2"].size)
            e2, p2 = pf["elem2"].astype(np.int64), pf["pos2"].astype(np.int64)
            np.testing.assert_array_equal(p2, 1 - prim_pos[e2])
            np.testing.assert_array_equal(pf["slotpos"][e2], k)       # one secondary per element
            np.testing.assert_array_equal(pf["ppos1"], prim_pos[pf["elem1"]])
            for which, sel in ((1, lambda e, a: a == prim_pos[e]), (2, lambda e, a: a != prim_pos[e])):
                o, el, t1 = pf[f"off{which}"], pf[f"elem{which}"], pf[f"tl{which}"]
                for r in range(pf[f"n{which}"]):
                    es = el[o[r]:o[r + 1]].tolist()
                    assert es == sorted(es)
                    assert es == [e for e, a in want.get(int(t1[r]), []) if sel(e, a)]
                    assert es                                     # only targets that have any
            # hub rows: split rows concatenate, in row order, to each target's list
            ps = pfold_lists_host(h["host"], hub_row=hub_row)
            for which in (1, 2):
                o, el, t1, seg = ps[f"off{which}"], ps[f"elem{which}"], ps[f"tl{which}"], ps[f"seg{which}"]
                assert ps[f"n{which}"] == o.size - 1 and np.all(np.diff(o) <= hub_row)
                np.testing.assert_array_equal(el, pf[f"elem{which}"])
                if seg is None:
                    continue
                assert sorted(seg[seg >= 0].tolist()) == list(range(ps[f"nslots{which}"]))
                for q, t in enumerate(ps[f"hub{which}_tl"]):
                    rows = np.flatnonzero((t1 == t) & (seg >= 0))
                    assert seg[rows].tolist() == list(range(ps[f"hub{which}_off"][q],
                                                            ps[f"hub{which}_off"][q + 1]))
                    assert np.all(seg[t1 == t] >= 0)


def test_pfold_element_records_hold_each_arguments_map_entry():
    """pfold pass-1 records: record column of every indirect argument holds
    the map entry that argument reads for the incidence's element; arguments
    on one (map, column) share a record column."""
    from paper_1403_7209_b200.device import gather_lists_host, pfold_lists_host, pfold_records_host
    mesh = apps.gen_hex_mesh(6, seed=1)
    prog, _ = apps.build_hydra_proxy(mesh, steps=1, seed=1)
    for loop in (prog[2], prog[3], prog[4]):
        h = gather_lists_host(loop, loop.iter_set.size, hubs=False)
        pf = pfold_lists_host(h["host"])
        rec, rcol = pfold_records_host(loop, pf["elem1"])
        assert rec.shape == (pf["elem1"].size, 2)                # edge_nodes columns 1 and 2
        for i, a in enumerate(loop.args):
            if a.kind != "indirect":
                assert rcol[i] == -1
                continue
            np.testing.assert_array_equal(rec[:, rcol[i]], a.map.table[pf["elem1"], a.slot])
        assert len({rcol[i] for i, a in enumerate(loop.args) if a.kind == "indirect"}) == 2
