"""Generate golden vectors by running the REFERENCE package (meshloop).

Run in the build container, where the reference is importable:

    PYTHONPATH=/root/reference/pkg/src python tests/golden/make_golden.py

It writes ``plans.npz``, ``renumber.npz``, ``partition.npz``, ``exec.npz``
and ``bytes.json`` next to this script.  Tests never import the reference:
they compare the oracle (``oracle/``) and the GPU backend against these
committed fixtures.  Meshes built here with the reference's own generators
are rebuilt in the tests with the product's generators, which pins those
too.  New meshes (3-D grids, the Hydra proxy) are built with the product
and converted into reference objects before the reference executes them.
"""
from __future__ import annotations

import json
import os
import sys
from pathlib import Path

import numpy as np

HERE = Path(__file__).resolve().parent
sys.path.insert(0, str(HERE.parent.parent))
sys.path.insert(0, os.environ.get("MESHLOOP_REF", "/root/reference/pkg/src"))

import meshloop as R                                   # noqa: E402  (the reference)
from meshloop import apps as RA                         # noqa: E402
from meshloop.plan import build_plan as ref_build_plan  # noqa: E402

from paper_1403_7209_b200 import apps as PA             # noqa: E402


# -- shared case builders (mirrored in tests/_cases.py with the product API) ------

def random_loop_mesh(api, rng, max_elems=500):
    """reference tests/conftest.py:59-79 with an injectable API module."""
    nt = int(rng.integers(2, max(3, max_elems // 3)))
    ni = int(rng.integers(1, max(2, max_elems - nt)))
    arity = int(rng.integers(1, 4))
    mesh = api.Mesh()
    tgt = mesh.decl_set("tgt", nt)
    it = mesh.decl_set("it", ni)
    m = mesh.decl_map("m", it, tgt, arity, rng.integers(1, nt + 1, size=ni * arity))
    vals = mesh.decl_dat("vals", tgt, 1, "int64", np.zeros(nt, dtype=np.int64))
    src = mesh.decl_dat("src", it, 1, "int64", rng.integers(0, 100, size=ni).astype(np.int64))
    args = [api.arg_direct(src, api.READ)] + [api.arg_indirect(vals, m, k + 1, api.INC)
                                              for k in range(arity)]

    def kern(s, *targets):
        for t in targets:
            t[0] += s[0]
    return mesh, api.Loop("fuzz", it, args, kern)


def mixmax_case(api):
    """reference tests/test_executor.py:367-394."""
    mesh = api.Mesh()
    nodes = mesh.decl_set("nodes", 30)
    edges = mesh.decl_set("edges", 60)
    rng = np.random.default_rng(7)
    en = mesh.decl_map("en", edges, nodes, 2, rng.integers(1, 31, 120))
    wide = mesh.decl_dat("wide", nodes, 5, "int64", rng.integers(-9, 9, 150))
    acc = mesh.decl_dat("acc", nodes, 5, "int64", np.zeros(150, np.int64))
    lo, hi, scale = api.Global(np.int64(10 ** 9)), api.Global(np.int64(-10 ** 9)), api.Global(np.int64(3))

    def kern(w1, w2, a1, a2, s, lo_, hi_):
        a1[:] += w2 * s[0]
        a2[:] += w1 * s[0]
        m, big = int(min(w1.min(), w2.min())), int(max(w1.max(), w2.max()))
        if m < lo_[0]:
            lo_[0] = m
        if big > hi_[0]:
            hi_[0] = big
    loop = api.Loop("mixmax", edges, [
        api.arg_indirect(wide, en, 1, api.READ), api.arg_indirect(wide, en, 2, api.READ),
        api.arg_indirect(acc, en, 1, api.INC), api.arg_indirect(acc, en, 2, api.INC),
        api.arg_global(scale, api.READ), api.arg_global(lo, api.MIN), api.arg_global(hi, api.MAX),
    ], kern)
    return mesh, loop, acc, lo, hi


def to_reference(mesh, program):
    """Convert a product mesh + program into reference objects (same data)."""
    rm = R.Mesh(auto_soa_threshold=None)
    sets = {n: rm.decl_set(n, s.size) for n, s in mesh.sets.items()}
    for n, m in mesh.maps.items():
        rm.decl_map(n, sets[m.from_set.name], sets[m.to_set.name], m.arity, (m.table + 1).ravel())
    for n, d in mesh.dats.items():
        rd = rm.decl_dat(n, sets[d.set.name], d.dim, d.dtype.name, d.fetch().ravel())
        if d.layout.name == "SOA":
            R.transform_layout(rd, R.SOA)
    gmap = {}
    loops = []
    for l in program:
        args = []
        for a in l.args:
            mode = getattr(R, a.mode.name)
            if a.kind == "global":
                g = gmap.setdefault(id(a.glob), R.Global(a.glob.buffer.copy(), name=a.glob.name))
                args.append(R.arg_global(g, mode))
            elif a.kind == "direct":
                args.append(R.arg_direct(rm.dats[a.dat.name], mode))
            else:
                args.append(R.arg_indirect(rm.dats[a.dat.name], rm.maps[a.map.name], a.slot + 1, mode))
        loops.append(R.Loop(l.name, sets[l.iter_set.name], args, l.kernel))
    return rm, loops, gmap


# -- plans ----------------------------------------------------------------------------

def plan_cases():
    cases = []
    clique = R.Mesh()
    nd = clique.decl_set("nodes", 1)
    ed = clique.decl_set("edges", 3)
    clique.decl_map("en", ed, nd, 1, [1, 1, 1])
    for bs in (1, 8):
        cases.append((f"clique_bs{bs}", 3, [("acc", np.zeros(3, np.int64))], bs))
    sm = RA.sample_mesh()
    cn = sm.maps["cell_nodes"].table
    for bs in (1, 4, 16):
        cases.append((f"sample_bs{bs}", 17, [("acc", cn[:, k]) for k in range(3)], bs))
    g16 = RA.gen_mesh(16)
    en = g16.maps["edge_nodes"].table
    for bs in (64, 128, 256, 512):
        cases.append((f"gen16_bs{bs}", en.shape[0], [("acc", en[:, 0]), ("acc", en[:, 1])], bs))
    g64 = RA.gen_mesh(64)
    en = g64.maps["edge_nodes"].table
    for bs in (64, 256, 2048):
        cases.append((f"gen64_bs{bs}", en.shape[0], [("flux", en[:, 0]), ("flux", en[:, 1])], bs))
    # offset-aliasing quirk (plan.py:77-81): second column of dat a exceeds the first
    # a's width is 2 (max of its FIRST column + 1), so a's second column [2, 3]
    # aliases b's ids [2, 3]: no real conflict, yet two block colours
    cases.append(("alias_quirk", 2, [("a", np.array([0, 1])), ("a", np.array([2, 3])),
                                     ("b", np.array([1, 0]))], 1))
    cases.append(("two_dats", 4, [("a", np.arange(4)), ("b", np.arange(4))], 1))
    cases.append(("empty", 0, [("acc", np.zeros(0, np.int64))], 16))
    cases.append(("direct_only", 20, [], 4))
    rng = np.random.default_rng(1234)
    for i in range(12):
        mesh, loop = random_loop_mesh(R, rng, max_elems=400)
        bs = int(rng.choice([1, 3, 7, 16, 64]))
        cols = [(a.dat.name, a.map.table[:, a.slot]) for a in loop.indirect_write_args()]
        cases.append((f"fuzz{i}_bs{bs}", loop.iter_set.size, cols, bs))
    # many colours: randomly numbered 3-D grid (SURVEY probe 4 shape, small)
    hexm = PA.gen_hex_mesh(10)
    PA.shuffle_mesh(hexm, seed=3)
    en = hexm.maps["edge_nodes"].table
    for bs in (32, 256):
        cases.append((f"hexshuf_bs{bs}", en.shape[0], [("res", en[:, 0]), ("res", en[:, 1])], bs))
    # hub nodes: element colours > 64 inside a block
    hub = PA.gen_hub_mesh(500, 3000, n_hubs=1, hub_share=0.5, seed=5)
    en = hub.maps["edge_nodes"].table
    cases.append(("hub_bs256", en.shape[0], [("res", en[:, 0]), ("res", en[:, 1])], 256))
    # ... and block colours > 64 (almost every block touches the hub)
    cases.append(("hub_bs4", en.shape[0], [("res", en[:, 0]), ("res", en[:, 1])], 4))
    return cases


def make_plans(out):
    index = []
    for name, n, cols, bs in plan_cases():
        p = ref_build_plan(n, [(k, np.asarray(c, np.int64)) for k, c in cols], bs)
        index.append({"name": name, "n": int(n), "bs": int(bs), "keys": [k for k, _ in cols]})
        for j, (_, c) in enumerate(cols):
            out[f"plan/{name}/col{j}"] = np.asarray(c, np.int64)
        out[f"plan/{name}/block_color"] = p.block_color
        out[f"plan/{name}/elem_color"] = p.elem_color
        out[f"plan/{name}/elem_ncolors"] = p.elem_ncolors
        out[f"plan/{name}/blocks_by_color"] = (np.concatenate(p.blocks_by_color)
                                               if p.ncolors else np.zeros(0, np.int64))
        out[f"plan/{name}/bpc"] = np.array([len(b) for b in p.blocks_by_color], np.int64)
        out[f"plan/{name}/block_elem_order"] = (np.concatenate(p.block_elem_order)
                                                if p.nblocks else np.zeros(0, np.int64))
        out[f"plan/{name}/ncolors"] = np.array(p.ncolors)
    return index


# -- renumbering ---------------------------------------------------------------------------

def path_mesh(order=(1, 2, 3, 4)):
    """reference tests/conftest.py:26-40."""
    mesh = R.Mesh()
    nodes = mesh.decl_set("nodes", 4)
    edges = mesh.decl_set("edges", 3)
    rows = []
    for k in range(3):
        rows.extend((order[k], order[k + 1]))
    mesh.decl_map("edge_nodes", edges, nodes, 2, rows)
    return mesh


def make_renumber(out):
    index = []
    meshes = [("path", path_mesh()), ("path_scrambled", path_mesh((3, 1, 4, 2))),
              ("sample", RA.sample_mesh()), ("gen5", RA.gen_mesh(5)), ("gen12", RA.gen_mesh(12))]
    # shuffled gen_mesh(12), shuffled with the reference itself
    sh = RA.gen_mesh(12)
    rng = np.random.default_rng(99)
    for s in ("nodes", "edges"):
        f = rng.permutation(sh.sets[s].size)
        R.apply_permutation(sh, R.Permutation(s, f, np.argsort(f), sh.version))
    meshes.append(("gen12_shuffled", sh))
    for name, mesh in meshes:
        tables = {n: m.table.copy() for n, m in mesh.maps.items()}
        perm = R.compute_ordering(mesh, mesh.sets["nodes"])
        out[f"ren/{name}/cm_forward"] = perm.forward
        for n, t in tables.items():
            out[f"ren/{name}/table/{n}"] = t
        rep = R.renumber_mesh(mesh)
        for s, p in rep["permutations"].items():
            out[f"ren/{name}/full/{s}"] = p.forward
        for n, (b, a) in rep["maps"].items():
            out[f"ren/{name}/span/{n}"] = np.array([b.max_span, b.mean_span, a.max_span, a.mean_span])
        index.append({"name": name, "sets": {n: s.size for n, s in mesh.sets.items()},
                      "maps": [[n, m.from_set.name, m.to_set.name, m.arity]
                               for n, m in mesh.maps.items()],
                      "perm_sets": list(rep["permutations"])})
    # product 3-D grid, shuffled by the product then renumbered by the reference
    hexm = PA.gen_hex_mesh(7)
    PA.shuffle_mesh(hexm, seed=11)
    prog = []
    rm, _, _ = to_reference(hexm, prog)
    for n, m in rm.maps.items():
        out[f"ren/hex7_shuffled/table/{n}"] = m.table.copy()
    rep = R.renumber_mesh(rm)
    for s, p in rep["permutations"].items():
        out[f"ren/hex7_shuffled/full/{s}"] = p.forward
    index.append({"name": "hex7_shuffled", "sets": {n: s.size for n, s in rm.sets.items()},
                  "maps": [[n, m.from_set.name, m.to_set.name, m.arity] for n, m in rm.maps.items()],
                  "perm_sets": list(rep["permutations"])})
    return index


# -- partitions and halos ---------------------------------------------------------------

def _dump_layout(out, key, layout):
    for sname, per in layout.sets.items():
        for r, h in enumerate(per):
            out[f"{key}/{sname}/{r}/owned"] = h.owned
            out[f"{key}/{sname}/{r}/exec"] = h.exec_halo
            out[f"{key}/{sname}/{r}/nonexec"] = h.nonexec_halo
            for src, ids in h.imports.items():
                out[f"{key}/{sname}/{r}/imp{src}"] = ids
            for dst, ids in h.exports.items():
                out[f"{key}/{sname}/{r}/exp{dst}"] = ids


def make_partition(out):
    index = []
    rng = np.random.default_rng(2024)
    pts = {"rand64_2d": rng.random((64, 2)), "rand50_2d_tie": rng.random((50, 2)),
           "rand200_3d": rng.random((200, 3))}
    pts["rand50_2d_tie"][10] = pts["rand50_2d_tie"][11]
    for name, xy in pts.items():
        m = R.Mesh()
        s = m.decl_set("pts", xy.shape[0])
        c = m.decl_dat("coords", s, xy.shape[1], "float64", xy.ravel())
        out[f"part/{name}/xy"] = xy
        for nr in (2, 4, 8):
            out[f"part/{name}/rcb{nr}"] = R.partition_rcb(c, nr).rank_of
    for size, nr in ((17, 2), (14, 1), (4, 8), (1001, 8)):
        out[f"part/trivial_{size}_{nr}"] = R.partition_trivial(R.Mesh().decl_set("s", size), nr).rank_of
    # layouts for whole programs, reference executor.build_layout
    from meshloop.executor import build_layout
    cases = []
    for nr, part in ((2, "trivial"), (4, "rcb"), (8, "rcb"), (3, "trivial")):
        cases.append((f"gen8_cellarea_{part}{nr}", "cell-area", 8, nr, part))
    for nr, part in ((2, "rcb"), (4, "trivial"), (4, "rcb")):
        cases.append((f"gen6_diffusion_{part}{nr}", "diffusion", 6, nr, part))
    for name, app, n, nr, part in cases:
        mesh = RA.gen_mesh(n)
        prog = (RA.build_cell_area(mesh, "int64")[0] if app == "cell-area"
                else RA.build_diffusion(mesh, 1, dtype="int64")[0])
        lay = build_layout(mesh, prog, R.BackendConfig(backend="ranks", nranks=nr, partitioner=part))
        _dump_layout(out, f"lay/{name}", lay)
        index.append({"name": name, "app": app, "n": n, "nranks": nr, "partitioner": part,
                      "sets": list(lay.sets)})
    # random fuzz meshes with trivial target partition (reference test_partition.py:145-152)
    rng = np.random.default_rng(77)
    for i in range(8):
        mesh, loop = random_loop_mesh(R, rng, max_elems=150)
        nr = int(rng.integers(2, 5))
        base = {"tgt": R.partition_trivial(mesh.sets["tgt"], nr)}
        asg = R.derive_assignments(mesh, [loop], base, nr)
        lay = R.build_halos(mesh, [loop], asg)
        out[f"fuzzlay/{i}/table"] = mesh.maps["m"].table
        _dump_layout(out, f"lay/fuzz{i}", lay)
        index.append({"name": f"fuzz{i}", "app": "fuzz", "nranks": nr,
                      "sizes": [mesh.sets["tgt"].size, mesh.sets["it"].size],
                      "sets": list(lay.sets)})
    return index


# -- executor results (reference run_serial / run_program) ---------------------------------

def make_exec(out):
    index = []
    # reference apps on reference meshes
    for app, n, dtype, steps in (("diffusion", 8, "int64", 3), ("diffusion", 8, "float64", 3),
                                 ("diffusion", 13, "float64", 2), ("cell-area", 6, "int64", 0),
                                 ("cell-area", 6, "float64", 0), ("cell-area", 0, "float64", 0)):
        mesh = RA.sample_mesh() if n == 0 else RA.gen_mesh(n)
        if app == "diffusion":
            prog, h = RA.build_diffusion(mesh, steps, dtype=dtype)
            R.run_program(prog, mesh, R.BackendConfig())
            res = {"u": h["u"].fetch(), "flux": h["flux"].fetch(),
                   "residuals": np.array([g.value for g in h["residuals"]])}
        else:
            prog, h = RA.build_cell_area(mesh, dtype)
            R.run_program(prog, mesh, R.BackendConfig())
            res = {"arean": h["arean"].fetch(), "areac": h["areac"].fetch(),
                   "total": np.atleast_1d(h["total"].value)}
        name = f"{app}_n{n}_{dtype}_s{steps}"
        for k, v in res.items():
            out[f"exec/{name}/{k}"] = np.asarray(v)
        index.append({"name": name, "app": app, "n": n, "dtype": dtype, "steps": steps})
    # renumbered diffusion (reference acceptance criterion 4 shape, small)
    mesh = RA.gen_mesh(10)
    prog, h = RA.build_diffusion(mesh, 2, dtype="int64")
    R.renumber_mesh(mesh)
    R.run_program(prog, mesh, R.BackendConfig())
    out["exec/diffusion_renum_n10_int64/u"] = h["u"].fetch()
    index.append({"name": "diffusion_renum_n10_int64", "app": "diffusion-renumbered"})
    # mixmax
    mesh, loop, acc, lo, hi = mixmax_case(R)
    R.run_serial(loop, mesh)
    out["exec/mixmax/acc"] = acc.fetch()
    out["exec/mixmax/lohi"] = np.array([lo.value, hi.value])
    index.append({"name": "mixmax", "app": "mixmax"})
    # fuzz
    rng = np.random.default_rng(31337)
    for i in range(6):
        seed = int(rng.integers(0, 2 ** 31))
        mesh, loop = random_loop_mesh(R, np.random.default_rng(seed), max_elems=300)
        R.run_serial(loop, mesh)
        out[f"exec/fuzz{i}/vals"] = mesh.dats["vals"].fetch()
        index.append({"name": f"fuzz{i}", "app": "fuzz", "seed": seed})
    # Hydra proxy on a small 3-D grid (product builder, reference executor)
    for N_, steps in ((5, 2), (7, 1)):
        pm = PA.gen_hex_mesh(N_, seed=4)
        prog, h = PA.build_hydra_proxy(pm, steps=steps, seed=4)
        rm, rloops, gmap = to_reference(pm, prog)
        R.run_program(rloops, rm, R.BackendConfig())
        name = f"proxy_hex{N_}_s{steps}"
        for k in ("q", "q_old", "res", "grad", "dt_loc"):
            out[f"exec/{name}/{k}"] = rm.dats[k].fetch()
        out[f"exec/{name}/rms"] = np.array([gmap[id(g)].value for g in h["rms"]])
        out[f"exec/{name}/dt_min"] = np.array([gmap[id(g)].value for g in h["dt_min"]])
        index.append({"name": name, "app": "proxy", "N": N_, "steps": steps})
    return index


def make_bytes():
    res = {}
    sm = RA.sample_mesh()
    prog, _ = RA.build_cell_area(sm, "int64")
    res["sample_cellarea_int64"] = {l.name: R.useful_bytes(l) for l in prog}
    g = RA.gen_mesh(64)
    prog, _ = RA.build_diffusion(g, 1)
    res["gen64_diffusion"] = {l.name: R.useful_bytes(l) for l in prog}
    pm = PA.gen_hex_mesh(12, seed=1)
    prog, _ = PA.build_hydra_proxy(pm, steps=1)
    rm, rloops, _ = to_reference(pm, prog)
    res["hex12_proxy"] = {l.name: R.useful_bytes(l) for l in rloops}
    return res


MESHIO_BAD = [
    "sets", "nope 1", "sets 1\nn x", "sets 1\nn 2\nmaps 1\nm n n 1\n1\n3\ndats 0",
    "sets 1\nn 1\nmaps 0\ndats 1\nd n 1 float64\nz",
    "sets 1\nn 1\nmaps 0\ndats 1\nd n 1 float16\n1", "sets 0\nmaps 0\ndats 0\nextra",
    "sets 1\nn 2\nmaps 1\nm n missing 1\n1\n2\ndats 0",
    "sets 1\nn 2\nmaps 1\nm n n 1\n1\n1.5\ndats 0",
    "sets 1\nn 3\nmaps 1\nm n n 1\n1 x", "sets 1\nn 3\nmaps 1\nm n n 1\n1 2",
    "sets 1\nn 2\nmaps 0\ndats 1\nd n 2 int64\n1 2 3.5 4",
    "sets 1\nn 2\nmaps 0\ndats 1\nd n 1 float64\n1e3",
    "sets 2\nn 2\nn 3\nmaps 0\ndats 0", "sets 1\nn 2\nmaps 1\nm n n 0\ndats 0",
    "sets 1\nn -1\nmaps 0\ndats 0",
]


def make_meshio():
    """Reference text form of two meshes and its error message per malformed input."""
    texts = {"sample": R.format_mesh(RA.sample_mesh()), "gen3": R.format_mesh(RA.gen_mesh(3))}
    errors = []
    for bad in MESHIO_BAD:
        try:
            R.parse_mesh(bad)
            errors.append([bad, None])
        except R.FormatError as err:
            errors.append([bad, str(err)])
    return {"texts": texts, "errors": errors}


def main():
    if sys.argv[1:] == ["meshio"]:
        (HERE / "meshio.json").write_text(json.dumps(make_meshio(), indent=1) + "\n")
        return
    (HERE / "meshio.json").write_text(json.dumps(make_meshio(), indent=1) + "\n")
    for fname, maker in (("plans.npz", make_plans), ("renumber.npz", make_renumber),
                         ("partition.npz", make_partition), ("exec.npz", make_exec)):
        out: dict = {}
        index = maker(out)
        out["__index__"] = np.frombuffer(json.dumps(index).encode(), dtype=np.uint8)
        np.savez_compressed(HERE / fname, **out)
        print(f"{fname}: {len(out)} arrays, {(HERE / fname).stat().st_size} bytes")
    (HERE / "bytes.json").write_text(json.dumps(make_bytes(), indent=1, sort_keys=True) + "\n")
    (HERE / "SOURCE.txt").write_text(
        "Generated by tests/golden/make_golden.py from the reference package meshloop "
        f"{R.__version__} at /root/reference/pkg/src (numpy {np.__version__}).\n")


if __name__ == "__main__":
    main()
