"""The C-ABI library loads on a CPU box and exports every symbol the public
header declares (no device calls here)."""
from __future__ import annotations

import ctypes as C
import re
import subprocess
from pathlib import Path

from paper_1403_7209_b200 import _native as N

HEADER = Path(__file__).resolve().parent.parent / "include" / "meshloop_b200.h"


def declared_functions() -> list[str]:
    text = HEADER.read_text()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"\b(ml_[a-z0-9_]+)\s*\(", text)))


def test_header_declares_what_the_binding_exports():
    assert declared_functions() == sorted(N.EXPORTED)


def test_library_loads_and_exports_every_declared_symbol():
    lib = N.lib()
    for name in declared_functions():
        assert hasattr(lib, name), name
    out = subprocess.run(["nm", "-D", "--defined-only", str(N.lib_path())], capture_output=True,
                         text=True, check=True).stdout
    exported = set(re.findall(r"\bT (ml_[a-z0-9_]+)$", out, flags=re.M))
    assert set(declared_functions()) <= exported


def test_library_is_built_for_sm100a_only():
    out = subprocess.run(["cuobjdump", "--list-elf", str(N.lib_path())], capture_output=True,
                         text=True).stdout
    archs = set(re.findall(r"sm_(\d+a?)", out))
    assert archs == {"100a"}, archs


def test_functor_registry_and_signatures():
    table = N.functor_table()
    names = {n for n, _ in table}
    for want in ("edge_flux", "copy", "diffusion_update", "boundary_fix", "tri_area",
                 "distribute", "distribute_int", "sum", "proxy_vflux", "proxy_iflux",
                 "proxy_grad", "proxy_update", "proxy_dt", "proxy_bc", "proxy_save", "mixmax"):
        assert want in names, want
    fid = C.c_int32()
    assert N.lib().ml_functor_lookup(b"proxy_vflux", N.ML_F64, C.byref(fid)) == 0
    nargs = C.c_int32()
    kinds, modes, dims, dts = [(C.c_int32 * 16)() for _ in range(4)]
    assert N.lib().ml_functor_signature(fid.value, C.byref(nargs), kinds, modes, dims, dts) == 0
    assert nargs.value == 11
    assert [dims[i] for i in range(11)] == [3, 6, 6, 18, 18, 3, 3, 19, 19, 6, 6]
    assert sum(dims[i] for i in range(1, 9)) == 92          # vfluxedge: 92 indirect doubles read
    assert N.lib().ml_functor_lookup(b"nope", 0, C.byref(fid)) != 0
    assert b"nope" in N.lib().ml_last_error()


def test_device_calls_fail_cleanly_without_init():
    p = C.c_void_p()
    rc = N.lib().ml_alloc(16, C.byref(p))
    assert rc != 0 and b"ml_init" in N.lib().ml_last_error()


def test_segmented_layout_range_matches_the_build():
    """The host decides which SOA dats get segmented (AoSoA) device copies
    from the range the library was built with (ml_seg_params), so the LP = 1
    kernels' compile-time layout classes and the mirrors agree."""
    import paper_1403_7209_b200 as ml
    from paper_1403_7209_b200.device import segmented
    shift, pad, mx, mn = N.seg_params()
    assert 1 <= shift <= 30 and pad >= 0 and mn >= 2
    mesh = ml.Mesh()
    nodes = mesh.decl_set("nodes", 10)
    for dim in (1, 3, 5, 6, 8, 18, 19, 24):
        d = mesh.decl_dat(f"d{dim}", nodes, dim, "float64", [0.0] * (10 * dim))
        assert segmented(d) == (d.layout is ml.SOA and dim > 1 and mn <= dim <= mx), dim
    aos = mesh.decl_dat("aos19", nodes, 19, "float64", [0.0] * 190)
    ml.transform_layout(aos, ml.AOS)
    assert not segmented(aos)


def test_hot_kernels_keep_two_ctas_per_sm():
    """Occupancy contract of the two latency-bound edge kernels: at <= 128
    registers per thread two 256-thread CTAs fit an SM (16 warps).  Above it
    they drop to one CTA and the fused flux loop runs ~20 % slower (DESIGN
    §7, register budget), so a code change that crosses it should fail here
    rather than in the bench."""
    import shutil
    exe = shutil.which("cuobjdump") or "/usr/local/cuda/bin/cuobjdump"
    out = subprocess.run([exe, "-res-usage", str(N.lib_path())], capture_output=True, text=True).stdout
    regs = {}
    lines = out.splitlines()
    for i, line in enumerate(lines):
        m = re.search(r"Function (\S+):", line)
        if m and i + 1 < len(lines):
            r = re.search(r"REG:(\d+)", lines[i + 1])
            if r:
                regs[m.group(1)] = int(r.group(1))
    # the compile-time-layout (LP = 1) instantiations the benchmark runs
    hot = {k: v for k, v in regs.items() if ("Li1EEEv" in k or "Li2EEEv" in k) and (
           ("k_pfold1" in k and "ProxyFluxes" in k) or ("k_gather" in k and "ProxyGrad" in k))}
    assert len(hot) >= 2, sorted(regs)[:5]
    assert all(v <= 128 for v in hot.values()), hot


def test_functor_record_columns_trait():
    """ml_functor_rec_cols: the proxy's grad functor declares (w, then node 1 /
    node 2 pairs); a functor without the trait declares none."""
    import ctypes as C

    def cols(name, dtype=N.ML_F64):
        fid, n = C.c_int32(), C.c_int32()
        N.check(N.lib().ml_functor_lookup(name.encode(), dtype, C.byref(fid)))
        buf = (C.c_int8 * 64)()
        N.check(N.lib().ml_functor_rec_cols(fid.value, buf, C.byref(n)))
        return list(buf[:n.value])
    assert cols("proxy_grad") == [-1, 0, 1, 0, 1, 0, 1]
    assert cols("proxy_bc") == [0, 1, 0, 1]
    assert cols("proxy_update") == []
