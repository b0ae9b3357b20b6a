"""Loop chaining legality (chain.py) on CPU: which adjacent pairs fuse, the
fused argument list, and — through the serial oracle running the fused
Python kernel — that a chained program computes the unchained result within
the reference tolerance.  The device runs of chained loops are in
test_gpu_parity.py."""
from __future__ import annotations

import numpy as np
import pytest

from oracle import serial
from paper_1403_7209_b200 import apps
from paper_1403_7209_b200.chain import chain_lookup, chain_pair, chain_program
from paper_1403_7209_b200.core import INC, READ, RW, Loop, arg_global, arg_indirect, Global


def _proxy(N=5, steps=2, seed=3):
    mesh = apps.gen_hex_mesh(N, seed=seed)
    prog, h = apps.build_hydra_proxy(mesh, steps=steps, seed=seed)
    return mesh, prog, h


def test_registered_chain_and_argument_map():
    fused, apos, bpos = chain_lookup("proxy_iflux", "proxy_vflux")
    assert fused == "proxy_fluxes" and len(apos) == 9 and len(bpos) == 11
    assert sorted(set(apos) | set(bpos)) == list(range(13))
    assert chain_lookup("proxy_vflux", "proxy_iflux") is None
    assert chain_lookup("edge_flux", "proxy_vflux") is None


def test_proxy_program_chains_each_flux_pair():
    mesh, prog, h = _proxy()
    out = chain_program(prog, mesh)
    assert [l.name for l in out] == ["save+dt_calc", "grad_edge", "iflux+vflux", "update", "bc"] * 2
    assert chain_program(prog, mesh)[2] is out[2]           # cached: compiled programs stay valid
    fl = out[2]
    iflux, vflux = prog[3], prog[4]
    assert list(fl.args[:7]) == list(iflux.args[:7])
    assert [fl.args[i] for i in (7, 8, 9, 10)] == [vflux.args[i] for i in (3, 4, 7, 8)]
    assert [a.mode for a in fl.args[11:]] == [INC, INC] and fl.args[11].dat is h["res"]


def test_direct_chain_carries_constants_and_reductions():
    """save -> dt_calc: two direct loops, the second with a constant (cfl) and
    a MIN reduction, fuse; the MIN global must not appear in the first loop."""
    from paper_1403_7209_b200.chain import _hazard_free
    from paper_1403_7209_b200.kernels import resolve_kernel
    mesh, prog, h = _proxy()
    sd = chain_program(prog, mesh)[0]
    assert sd.name == "save+dt_calc" and len(sd.args) == 5
    b = resolve_kernel(sd.kernel)
    assert b.functor == "proxy_save_dt" and b.fconsts == resolve_kernel(prog[1].kernel).fconsts
    assert sd.args[4].glob is h["dt_min"][0]
    save, dt = prog[0], prog[1]
    assert _hazard_free(save, dt)
    reads_min = Loop("save", save.iter_set, list(save.args) + [arg_global(h["dt_min"][0], READ)],
                     save.kernel)
    assert not _hazard_free(reads_min, dt)                # dt_calc's MIN read by the other loop
    assert not _hazard_free(dt, reads_min)


def test_chained_program_matches_unchained_in_the_oracle():
    ma, pa, ha = _proxy(6, steps=2, seed=4)
    mb, pb, hb = _proxy(6, steps=2, seed=4)
    serial.run_program(pa)
    serial.run_program(chain_program(pb, mb))
    for k in ("q", "q_old", "dt_loc"):
        np.testing.assert_allclose(hb[k].fetch(), ha[k].fetch(), rtol=1e-12, atol=1e-300)
    assert [g.value for g in hb["dt_min"]] == [g.value for g in ha["dt_min"]]
    ma, pa, ha = _proxy(6, steps=1, seed=4)
    mb, pb, hb = _proxy(6, steps=1, seed=4)
    serial.run_program(pa[:5])
    serial.run_program(chain_program(pb[:5], mb))
    ref = ha["res"].fetch()
    np.testing.assert_allclose(hb["res"].fetch(), ref, rtol=1e-12, atol=1e-12 * np.abs(ref).max())


@pytest.mark.parametrize("change", ["other_set", "reads_res", "writes_q", "global", "swapped"])
def test_illegal_pairs_do_not_chain(change):
    mesh, prog, h = _proxy(4, steps=1)
    iflux, vflux = prog[3], prog[4]
    args = list(vflux.args)
    en = iflux.args[1].map
    A, B = iflux, vflux
    if change == "other_set":
        B = Loop("vflux", mesh.sets["nodes"], [], vflux.kernel)
    elif change == "reads_res":          # the second loop READs what the first INCs
        args[1] = arg_indirect(h["res"], en, 1, READ)
        B = Loop("vflux", vflux.iter_set, args, vflux.kernel)
    elif change == "writes_q":           # the second loop modifies what the first reads
        args[1] = arg_indirect(h["q"], en, 1, RW)
        B = Loop("vflux", vflux.iter_set, args, vflux.kernel)
    elif change == "global":
        g = Global(np.zeros(1), "g")
        B = Loop("vflux", vflux.iter_set, args + [arg_global(g, INC)], vflux.kernel)
    elif change == "swapped":
        A, B = vflux, iflux
    assert chain_pair(A, B) is None
    assert [l.name for l in chain_program([A, B], mesh)] == [A.name, B.name]


def test_non_identical_shared_argument_does_not_chain():
    """vflux's x rows not listed in the fused map must equal iflux's exactly."""
    mesh, prog, h = _proxy(4, steps=1)
    iflux, vflux = prog[3], prog[4]
    args = list(vflux.args)
    args[5] = arg_indirect(h["x"], iflux.args[3].map, 2, READ)     # slot swapped
    assert chain_pair(iflux, Loop("vflux", vflux.iter_set, args, vflux.kernel)) is None


def test_auto_schedule_follows_measured_choices():
    """"auto" (the default INC schedule) resolves as the B200 measurements
    chose: pfold for the wide-gather flux loops (hub meshes included: pfold
    splits hub rows), gather for iflux, grad_edge and the diffusion edge flux."""
    from paper_1403_7209_b200.executor import auto_schedule
    mesh, prog, h = _proxy(6, steps=1)
    out = chain_program(prog, mesh)
    assert auto_schedule(prog[2]) == "gather"           # grad_edge: 16 read / 36 INC
    assert auto_schedule(prog[3]) == "gather"           # iflux: 34 / 10
    assert auto_schedule(prog[4]) == "pfold"            # vflux: 92 / 10
    assert auto_schedule(out[2]) == "pfold"             # iflux+vflux: 126 / 10
    assert auto_schedule(prog[6]) == "gather"           # bc: indirect WRITE
    d = apps.gen_mesh(20)
    dprog, _ = apps.build_diffusion(d, 1, dtype="float64")
    assert auto_schedule(dprog[1]) == "gather"
    hub = apps.gen_hub_mesh(2000, 20000, n_hubs=4, hub_share=0.2, seed=1)
    from paper_1403_7209_b200.core import Loop as L
    e = hub.sets["edges"]
    en = hub.maps["edge_nodes"]
    wide = hub.decl_dat("wide", hub.sets["nodes"], 8, "float64", np.zeros(hub.sets["nodes"].size * 8))
    acc = hub.decl_dat("acc1", hub.sets["nodes"], 1, "float64", np.zeros(hub.sets["nodes"].size))
    loop = L("wide", e, [arg_indirect(wide, en, 1, READ), arg_indirect(wide, en, 2, READ),
                         arg_indirect(acc, en, 1, INC), arg_indirect(acc, en, 2, INC)], lambda *a: None)
    assert auto_schedule(loop) == "pfold"               # 16 / 2, hub rows split


def test_chain_needs_the_fused_functor_for_the_loops_type():
    """The proxy chain is registered for float64 only: int64 copies of the
    same loops stay unchained (no missing-functor failure at compile time)."""
    from paper_1403_7209_b200 import _native as N
    import ctypes as C
    fid = C.c_int32()
    assert N.lib().ml_functor_lookup(b"proxy_fluxes", N.ML_I64, C.byref(fid)) != 0
    mesh, prog, h = _proxy(4, steps=1)
    iflux, vflux = prog[3], prog[4]
    ints = {}

    def as_int(a):
        if a.kind == "global":
            return a
        d = a.dat
        if d.name not in ints:
            ints[d.name] = mesh.decl_dat(d.name + "_i", d.set, d.dim, "int64",
                                         np.zeros(d.set.size * d.dim, np.int64))
        return (arg_indirect(ints[d.name], a.map, a.slot + 1, a.mode) if a.kind == "indirect"
                else type(a)("direct", a.mode, dat=ints[d.name]))
    A = Loop("iflux", iflux.iter_set, [as_int(a) for a in iflux.args], iflux.kernel)
    B = Loop("vflux", vflux.iter_set, [as_int(a) for a in vflux.args], vflux.kernel)
    assert chain_pair(iflux, vflux) is not None
    assert chain_pair(A, B) is None


def test_loops_named_by_a_per_loop_table_are_not_fused():
    """a block_size_table / inc_schedule_table entry for a member
    loop must apply to that loop, so the pair is left unfused."""
    from paper_1403_7209_b200.chain import chain_program
    mesh = apps.gen_hex_mesh(4, seed=1)
    prog, _h = apps.build_hydra_proxy(mesh, steps=1, seed=1)
    names = [l.name for l in chain_program(prog, mesh)]
    assert "iflux+vflux" in names
    for pinned in ({"vflux"}, {"iflux"}):
        names = [l.name for l in chain_program(prog, mesh, frozenset(pinned))]
        assert "iflux" in names and "vflux" in names and "iflux+vflux" not in names
