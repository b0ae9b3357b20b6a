"""Pin the CPU oracle to the reference: every oracle module must reproduce the
golden vectors the reference package produced (tests/golden/make_golden.py).
CPU only."""
from __future__ import annotations

import numpy as np
import pytest

from conftest import golden, golden_bytes
import _cases
from oracle import bulk, partition as opart, perf as operf, plan as oplan, renumber as oren
from oracle import serial as oserial
from paper_1403_7209_b200 import apps


# -- plans ------------------------------------------------------------------------------

def _plan_case(g, case):
    name = case["name"]
    cols = [(k, g[f"plan/{name}/col{j}"]) for j, k in enumerate(case["keys"])]
    return name, case["n"], cols, case["bs"]


def test_oracle_plan_matches_reference_golden():
    g = golden("plans.npz")
    assert len(g.index) >= 25
    for case in g.index:
        name, n, cols, bs = _plan_case(g, case)
        p = oplan.build_plan(n, cols if case["keys"] else [], bs)
        np.testing.assert_array_equal(p.block_color, g[f"plan/{name}/block_color"], name)
        np.testing.assert_array_equal(p.elem_color, g[f"plan/{name}/elem_color"], name)
        np.testing.assert_array_equal(p.elem_ncolors, g[f"plan/{name}/elem_ncolors"], name)
        assert p.ncolors == int(g[f"plan/{name}/ncolors"]), name
        flat = np.concatenate(p.blocks_by_color) if p.ncolors else np.zeros(0, np.int64)
        np.testing.assert_array_equal(flat, g[f"plan/{name}/blocks_by_color"], name)
        order = np.concatenate(p.block_elem_order) if p.nblocks else np.zeros(0, np.int64)
        np.testing.assert_array_equal(order, g[f"plan/{name}/block_elem_order"], name)


def test_golden_pins_the_offset_quirk_and_known_answers():
    g = golden("plans.npz")
    assert int(g["plan/alias_quirk/ncolors"]) == 2          # false conflict (plan.py:77-81)
    assert int(g["plan/two_dats/ncolors"]) == 1
    assert int(g["plan/clique_bs1/ncolors"]) == 3
    assert g["plan/clique_bs8/elem_ncolors"].tolist() == [3]
    assert int(g["plan/empty/ncolors"]) == 0
    assert int(g["plan/direct_only/ncolors"]) == 1
    assert g["plan/hub_bs256/elem_ncolors"].max() > 64     # spills past one colour word
    assert int(g["plan/hub_bs4/ncolors"]) > 64


# -- renumbering --------------------------------------------------------------------------

def _maps_of(g, case):
    name = case["name"]
    return [{"name": mn, "from": f, "to": t, "table": g[f"ren/{name}/table/{mn}"]}
            for mn, f, t, _a in case["maps"]]


def test_oracle_cm_ordering_matches_reference_golden():
    g = golden("renumber.npz")
    for case in g.index:
        name = case["name"]
        if f"ren/{name}/cm_forward" not in g:
            continue
        maps = _maps_of(g, case)
        order = oren.cm_order(oren.adjacency(maps, "nodes", case["sets"]["nodes"]))
        np.testing.assert_array_equal(oren.forward_of(order), g[f"ren/{name}/cm_forward"], name)


def test_oracle_full_renumber_matches_reference_golden():
    g = golden("renumber.npz")
    for case in g.index:
        name = case["name"]
        fwds, _, _ = oren.renumber(case["sets"], _maps_of(g, case), [])
        assert sorted(fwds) == sorted(case["perm_sets"]), name
        for s, f in fwds.items():
            np.testing.assert_array_equal(f, g[f"ren/{name}/full/{s}"], f"{name}/{s}")


def test_ordered_path_is_identity_not_reversed():
    g = golden("renumber.npz")
    assert g["ren/path/cm_forward"].tolist() == [0, 1, 2, 3]


# -- partitions and halos -------------------------------------------------------------------

def test_oracle_partitioners_match_reference_golden():
    g = golden("partition.npz")
    for name in ("rand64_2d", "rand50_2d_tie", "rand200_3d"):
        xy = g[f"part/{name}/xy"]
        for nr in (2, 4, 8):
            np.testing.assert_array_equal(opart.rcb(xy, nr), g[f"part/{name}/rcb{nr}"])
    for size, nr in ((17, 2), (14, 1), (4, 8), (1001, 8)):
        np.testing.assert_array_equal(opart.trivial(size, nr), g[f"part/trivial_{size}_{nr}"])


def _loops_as_arrays(program):
    out = []
    for l in program:
        args = []
        for a in l.args:
            if a.kind == "indirect":
                args.append(("indirect", a.mode.name, a.dat.set.name, a.map.table[:, a.slot],
                             a.map.table))
            elif a.kind == "direct":
                args.append(("direct", a.mode.name, a.dat.set.name, None, None))
        out.append({"iter": l.iter_set.name, "args": args})
    return out


def _check_layout(g, key, per_set):
    for sname, per in per_set.items():
        for r, (owned, ex, nx, imports, exports) in enumerate(per):
            np.testing.assert_array_equal(owned, g[f"{key}/{sname}/{r}/owned"], f"{key} {sname} {r}")
            np.testing.assert_array_equal(ex, g[f"{key}/{sname}/{r}/exec"], f"{key} {sname} {r}")
            np.testing.assert_array_equal(nx, g[f"{key}/{sname}/{r}/nonexec"], f"{key} {sname} {r}")
            want_imp = sorted(int(k.rsplit("imp", 1)[1]) for k in g.keys(f"{key}/{sname}/{r}/imp"))
            want_exp = sorted(int(k.rsplit("exp", 1)[1]) for k in g.keys(f"{key}/{sname}/{r}/exp"))
            assert sorted(imports) == want_imp and sorted(exports) == want_exp
            for q, ids in imports.items():
                np.testing.assert_array_equal(ids, g[f"{key}/{sname}/{r}/imp{q}"])
            for q, ids in exports.items():
                np.testing.assert_array_equal(ids, g[f"{key}/{sname}/{r}/exp{q}"])


def test_oracle_halos_match_reference_golden():
    g = golden("partition.npz")
    for case in g.index:
        name, nr = case["name"], case["nranks"]
        if case["app"] == "fuzz":
            nt, ni = case["sizes"]
            table = g[f"fuzzlay/{name[4:]}/table"]
            loops = [{"iter": "it", "args": [("direct", "READ", "it", None, None)]
                      + [("indirect", "INC", "tgt", table[:, k], table) for k in range(table.shape[1])]}]
            owner = opart.derive(loops, {"tgt": opart.trivial(nt, nr)}, {"tgt": nt, "it": ni}, nr)
        else:
            mesh, prog, _ = _cases.build_app(case["app"], case["n"], "int64", 1)
            loops = _loops_as_arrays(prog)
            targets = []
            for lp in loops:
                for a in lp["args"]:
                    if a[0] == "indirect" and a[2] not in targets:
                        targets.append(a[2])
            base = {}
            for t in targets:
                base[t] = (opart.rcb(mesh.dats["coords"].fetch(), nr) if case["partitioner"] == "rcb"
                           else opart.trivial(mesh.sets[t].size, nr))
            owner = opart.derive(loops, base, {n: s.size for n, s in mesh.sets.items()}, nr)
        _check_layout(g, f"lay/{name}", opart.halos(loops, owner, nr))


# -- executor semantics -------------------------------------------------------------------

def _exec_cases():
    return [c for c in golden("exec.npz").index if c["app"] in ("diffusion", "cell-area")]


@pytest.mark.parametrize("case", _exec_cases(), ids=lambda c: c["name"])
def test_oracle_serial_reproduces_reference_bit_for_bit(case):
    """The per-element oracle on the product's app programs == reference run_program."""
    g = golden("exec.npz")
    mesh, prog, h = _cases.build_app(case["app"], case["n"], case["dtype"], case["steps"])
    oserial.run_program(prog)
    for k, v in _cases.app_results(case["app"], h).items():
        np.testing.assert_array_equal(v, g[f"exec/{case['name']}/{k}"], k)


@pytest.mark.parametrize("case", _exec_cases(), ids=lambda c: c["name"])
def test_oracle_bulk_is_bit_identical_to_serial(case):
    g = golden("exec.npz")
    mesh, prog, h = _cases.build_app(case["app"], case["n"], case["dtype"], case["steps"])
    bulk.run_program(prog)
    for k, v in _cases.app_results(case["app"], h).items():
        np.testing.assert_array_equal(v, g[f"exec/{case['name']}/{k}"], k)


def test_oracle_renumbered_diffusion_matches_reference():
    g = golden("exec.npz")
    from paper_1403_7209_b200 import renumber_mesh
    mesh = apps.gen_mesh(10)
    prog, h = apps.build_diffusion(mesh, 2, dtype="int64")
    renumber_mesh(mesh)
    oserial.run_program(prog)
    np.testing.assert_array_equal(h["u"].fetch(), g["exec/diffusion_renum_n10_int64/u"])


def test_oracle_mixmax_and_fuzz_match_reference():
    g = golden("exec.npz")
    mesh, loop, acc, lo, hi = _cases.mixmax_case()
    oserial.run_loop(loop)
    np.testing.assert_array_equal(acc.fetch(), g["exec/mixmax/acc"])
    assert [lo.value, hi.value] == g["exec/mixmax/lohi"].tolist()
    for case in golden("exec.npz").index:
        if case["app"] != "fuzz":
            continue
        mesh, loop = _cases.random_loop_mesh(np.random.default_rng(case["seed"]), max_elems=300)
        oserial.run_loop(loop)
        np.testing.assert_array_equal(mesh.dats["vals"].fetch(), g[f"exec/{case['name']}/vals"])


@pytest.mark.parametrize("N,steps", [(5, 2), (7, 1)])
@pytest.mark.parametrize("which", ["serial", "bulk"])
def test_oracle_proxy_matches_reference(N, steps, which):
    g = golden("exec.npz")
    mesh = apps.gen_hex_mesh(N, seed=4)
    prog, h = apps.build_hydra_proxy(mesh, steps=steps, seed=4)
    if which == "serial":
        oserial.run_program(prog)
    else:
        bulk.run_program(prog)
    name = f"proxy_hex{N}_s{steps}"
    for k in ("q", "q_old", "res", "grad", "dt_loc"):
        np.testing.assert_array_equal(h[k].fetch(), g[f"exec/{name}/{k}"], k)
    np.testing.assert_array_equal([r.value for r in h["rms"]], g[f"exec/{name}/rms"])
    np.testing.assert_array_equal([r.value for r in h["dt_min"]], g[f"exec/{name}/dt_min"])


def test_oracle_coloured_schedule_matches_serial_on_int64():
    mesh, prog, h = _cases.build_app("diffusion", 8, "int64", 3)
    for loop in prog:
        p = oplan.build_plan(loop.iter_set.size, oplan.write_columns(loop), 16)
        oserial.run_loop_coloured(loop, p)
    g = golden("exec.npz")
    np.testing.assert_array_equal(h["u"].fetch(), g["exec/diffusion_n8_int64_s3/u"])


# -- bytes -------------------------------------------------------------------------------

def test_oracle_useful_bytes_match_reference():
    want = golden_bytes()
    m = apps.sample_mesh()
    prog, _ = apps.build_cell_area(m, "int64")
    assert {l.name: operf.useful_bytes(l) for l in prog} == want["sample_cellarea_int64"]
    m = apps.gen_mesh(64)
    prog, _ = apps.build_diffusion(m, 1)
    assert {l.name: operf.useful_bytes(l) for l in prog} == want["gen64_diffusion"]
    m = apps.gen_hex_mesh(12, seed=1)
    prog, _ = apps.build_hydra_proxy(m, steps=1)
    assert {l.name: operf.useful_bytes(l) for l in prog} == want["hex12_proxy"]
    assert want["sample_cellarea_int64"]["area_distribute"] == 360     # reference test_perf.py:258
