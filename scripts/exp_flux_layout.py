"""Experiment driver for scripts/exp_flux_layout.cu (not product code).

Builds the bench mesh (94^3, shuffled, CM-renumbered) and the primary-fold
lists of the fused iflux+vflux loop, runs the hand-written pass-1 kernel for
the SOA and AOSOA layouts, checks they agree bit for bit (same arithmetic),
and times each with CUDA events (mean of --reps launches after warm-up).

    python scripts/exp_flux_layout.py [--grid 94] [--reps 50]
"""
from __future__ import annotations

import argparse
import ctypes as C
import json
import sys
from pathlib import Path

import numpy as np
import torch

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))


def to_aosoa(v: np.ndarray) -> np.ndarray:
    """(n, D) logical -> flat AoSoA with 32-node blocks, padded to whole blocks."""
    n, D = v.shape
    nb = -(-n // 32)
    pad = np.zeros((nb * 32, D))
    pad[:n] = v
    return np.ascontiguousarray(pad.reshape(nb, 32, D).transpose(0, 2, 1)).reshape(-1)


def from_aosoa(f: np.ndarray, n: int, D: int) -> np.ndarray:
    nb = -(-n // 32)
    return f.reshape(nb, D, 32).transpose(0, 2, 1).reshape(nb * 32, D)[:n]


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--grid", type=int, default=94)
    ap.add_argument("--reps", type=int, default=50)
    ap.add_argument("--only", nargs="*", default=[], help="variant names to run (plus soa, the reference)")
    args = ap.parse_args()
    from paper_1403_7209_b200 import apps, renumber_mesh
    mesh = apps.gen_hex_mesh(args.grid, seed=0)
    apps.shuffle_mesh(mesh, seed=1)
    prog, h = apps.build_hydra_proxy(mesh, steps=1, seed=0)
    renumber_mesh(mesh)
    t = mesh.maps["edge_nodes"].table
    n, m = mesh.sets["nodes"].size, mesh.sets["edges"].size
    # primary-fold lists: pass-1 rows by first target, secondary slots by second
    o1 = np.lexsort((np.arange(m), t[:, 0]))
    c1 = np.bincount(t[:, 0], minlength=n)
    tl1 = np.flatnonzero(c1).astype(np.int32)
    off1 = np.concatenate([[0], np.cumsum(c1[tl1])]).astype(np.int32)
    elem1 = o1.astype(np.int32)
    rec = np.ascontiguousarray(t[elem1]).astype(np.int32)
    o2 = np.lexsort((np.arange(m), t[:, 1]))
    slotpos = np.empty(m, np.int32)
    slotpos[o2] = np.arange(m, dtype=np.int32)

    # warp tasks for the lane-per-edge kernel: consecutive rows packed greedily
    # while their primary edges fit in 32 lanes
    cnt = np.diff(off1)
    wrow = [0]
    acc = 0
    for r, c in enumerate(cnt):
        if acc + c > 32:
            wrow.append(r)
            acc = 0
        acc += c
    wrow.append(cnt.size)
    wrow = np.asarray(wrow, np.int32)
    # per-lane records of the warp tasks
    ntask = wrow.size - 1
    lrec = np.full((ntask, 32, 4), -1, np.int32)
    tmask = np.zeros(ntask, np.uint32)
    kk0 = off1[wrow[:-1]]
    for tsk in range(ntask):
        r0, r1_ = wrow[tsk], wrow[tsk + 1]
        b0, b1 = off1[r0], off1[r1_]
        ks = np.arange(b0, b1)
        e = elem1[ks]
        lrec[tsk, :ks.size] = np.stack([rec[ks, 0], rec[ks, 1], e, slotpos[e]], 1)
        tmask[tsk] = np.bitwise_or.reduce((1 << (off1[r0:r1_] - b0)).astype(np.uint32))
    # slot-major incidence lists (j-th primary incidence of row t at j * n1 + t)
    J = int(np.diff(off1).max())
    n1 = tl1.size
    cnt1 = np.diff(off1).astype(np.int32)
    elem_sm = np.zeros((J, n1), np.int32)
    rec_sm = np.zeros((J, 2, n1), np.int32)
    for j in range(J):
        has = cnt1 > j
        kk = off1[:-1][has] + j
        elem_sm[j, has] = elem1[kk]
        rec_sm[j, 0, has] = rec[kk, 0]
        rec_sm[j, 1, has] = rec[kk, 1]
    dev = torch.device("cuda")
    lib = C.CDLL(str(ROOT / "scripts" / "_exp_flux.so"))
    lib.exp_flux_run.argtypes = [C.c_int] + [C.c_void_p] * 13 + [C.c_int64, C.c_int64, C.c_int, C.c_void_p]
    lib.exp_flux_lanes.argtypes = ([C.c_int] + [C.c_void_p] * 13 + [C.c_int64, C.c_int64, C.c_void_p,
                                   C.c_int64, C.c_int, C.c_void_p])
    lib.exp_flux_lock.argtypes = [C.c_int] + [C.c_void_p] * 13 + [C.c_int64, C.c_int64, C.c_int, C.c_void_p]
    lib.exp_flux_reg.argtypes = [C.c_int] + [C.c_void_p] * 13 + [C.c_int64, C.c_int64, C.c_int, C.c_void_p]
    lib.exp_flux_h.argtypes = [C.c_int] + [C.c_void_p] * 13 + [C.c_int64, C.c_int64, C.c_int, C.c_void_p]
    lib.exp_flux_split.argtypes = [C.c_int] + [C.c_void_p] * 13 + [C.c_int64, C.c_int64, C.c_int, C.c_void_p]
    lib.exp_flux_sm.argtypes = ([C.c_int] + [C.c_void_p] * 10 + [C.c_int64, C.c_int64] + [C.c_void_p] * 3
                                + [C.c_int, C.c_void_p])
    lib.exp_flux_smrun.argtypes = [C.c_int] + [C.c_void_p] * 13 + [C.c_int64, C.c_int64, C.c_int, C.c_void_p]
    lib.exp_flux_pf.argtypes = [C.c_int] + [C.c_void_p] * 13 + [C.c_int64, C.c_int64, C.c_int, C.c_void_p]
    lib.exp_flux_bulk.argtypes = [C.c_int] + [C.c_void_p] * 13 + [C.c_int64, C.c_int64, C.c_int, C.c_void_p]
    lib.exp_flux_cpa.argtypes = [C.c_int] + [C.c_void_p] * 13 + [C.c_int64, C.c_int64, C.c_int, C.c_void_p]
    lib.exp_flux_own.argtypes = [C.c_int] + [C.c_void_p] * 13 + [C.c_int64, C.c_int64, C.c_int, C.c_void_p]
    lib.exp_flux_aos.argtypes = [C.c_int] + [C.c_void_p] * 13 + [C.c_int64, C.c_int64, C.c_int, C.c_void_p]
    lib.exp_flux_lrec.argtypes = ([C.c_int] + [C.c_void_p] * 8 + [C.c_int64, C.c_void_p, C.c_void_p,
                                  C.c_int64, C.c_int, C.c_void_p])
    vals = {k: h[k].fetch() for k in ("q", "x", "lim", "grad", "aux", "res", "w")}
    vals["grad"] = np.random.default_rng(0).random(vals["grad"].shape)   # nonzero gradients
    vals["res"] = np.random.default_rng(1).random(vals["res"].shape)
    ints = {k: torch.from_numpy(v).to(dev) for k, v in
            (("cnt1", cnt1), ("elem_sm", elem_sm.reshape(-1)), ("rec_sm", rec_sm.reshape(-1)),
             ("off1", off1), ("elem1", elem1), ("tl1", tl1), ("rec", rec.reshape(-1)), ("slotpos", slotpos),
             ("wrow", wrow), ("lrec", lrec.reshape(-1)), ("tmask", tmask.view(np.int32)))}
    sms = torch.cuda.get_device_properties(0).multi_processor_count
    out = {}
    results = {}
    for lay, lanes, name in ((0, 0, "soa"), (1, 0, "aosoa"), (0, 1, "soa_lanes"), (1, 1, "aosoa_lanes"),
                             (0, 2, "soa_lrec"), (1, 2, "aosoa_lrec"), (2, 0, "soa_128x5"),
                             (3, 0, "aosoa_128x5"), (0, 3, "soa_lock3"), (1, 3, "aosoa_lock3"),
                             (0, 4, "soa_lock2"), (1, 4, "aosoa_lock2"), (0, 5, "soa_lock4"),
                             (1, 5, "aosoa_lock4"), (0, 6, "soa_reg1"), (1, 6, "aosoa_reg1"),
                             (0, 7, "soa_reg2"), (1, 7, "aosoa_reg2"),
                             (0, 10, "soa_pf"), (1, 11, "aosoa_pf"), (0, 12, "soa_hint"), (1, 13, "aosoa_hint"),
                             (0, 14, "soa_hint_pf"), (1, 15, "aosoa_hint_pf"), (0, 16, "soa_nbr_noalloc"),
                             (1, 17, "aosoa_nbr_noalloc"), (0, 20, "soa_split2"), (1, 21, "aosoa_split2"),
                             (0, 22, "soa_split3"), (1, 23, "aosoa_split3"), (0, 24, "soa_split4"),
                             (1, 25, "aosoa_split4"), (4, 30, "aos_pad"), (4, 31, "aos_pad_128x5"),
                             (0, 40, "own0"), (0, 48, "own_aux"), (0, 44, "own_grad"), (0, 52, "own_grad_aux"),
                             (0, 55, "own_all"), (0, 60, "cpa_grad_aux"), (0, 61, "cpa_aux"),
                             (0, 62, "cpa_all"), (0, 63, "cpa_grad_aux_64x6"), (0, 64, "cpa_grad"),
                             (4, 70, "bulk_grad_aux"), (4, 71, "bulk_all_64x3"), (4, 72, "bulk_aux"),
                             (4, 73, "bulk_grad_aux_64x4"), (0, 80, "pf_soa_ga"), (1, 81, "pf_aosoa_ga"),
                             (1, 82, "pf_aosoa_all"), (0, 83, "pf_soa_all"), (1, 84, "pf_aosoa_none"),
                             (0, 90, "smrun_soa"), (1, 91, "smrun_aosoa"), (0, 100, "slotmajor_soa"),
                             (1, 101, "slotmajor_aosoa")):
        if args.only and name not in args.only and name != "soa":
            continue
        def put(k):
            v = vals[k]
            if k in ("x", "w"):
                return torch.from_numpy(np.ascontiguousarray(v).reshape(-1)).to(dev)
            if lay == 4:                      # padded AoS rows
                D = v.shape[1]
                pv = np.zeros((v.shape[0], (D + 1) // 2 * 2))
                pv[:, :D] = v
                return torch.from_numpy(pv.reshape(-1)).to(dev)
            if lay % 2 == 0:
                return torch.from_numpy(np.ascontiguousarray(v.T).reshape(-1)).to(dev)
            return torch.from_numpy(to_aosoa(v)).to(dev)
        T = {k: put(k) for k in vals}
        res0 = T["res"].clone()
        slots = torch.zeros(m * 6, dtype=torch.float64, device=dev)
        stream = torch.cuda.current_stream().cuda_stream

        def launch():
            common = (lay, T["w"].data_ptr(), T["q"].data_ptr(), T["x"].data_ptr(),
                      T["lim"].data_ptr(), T["grad"].data_ptr(), T["aux"].data_ptr(),
                      T["res"].data_ptr(), slots.data_ptr(), ints["off1"].data_ptr(),
                      ints["elem1"].data_ptr(), ints["tl1"].data_ptr(), ints["rec"].data_ptr(),
                      ints["slotpos"].data_ptr(), int(tl1.size), n)
            if lanes >= 100:
                rc = lib.exp_flux_sm(lay, T["w"].data_ptr(), T["q"].data_ptr(), T["x"].data_ptr(),
                                     T["lim"].data_ptr(), T["grad"].data_ptr(), T["aux"].data_ptr(),
                                     T["res"].data_ptr(), slots.data_ptr(), ints["tl1"].data_ptr(),
                                     ints["slotpos"].data_ptr(), int(tl1.size), n, ints["cnt1"].data_ptr(),
                                     ints["elem_sm"].data_ptr(), ints["rec_sm"].data_ptr(), sms, stream)
            elif lanes >= 90:
                rc = lib.exp_flux_smrun(lanes - 90, *common[1:], sms, stream)
            elif lanes >= 80:
                rc = lib.exp_flux_pf(lanes - 80, *common[1:], sms, stream)
            elif lanes >= 70:
                rc = lib.exp_flux_bulk(lanes - 70, *common[1:], sms, stream)
            elif lanes >= 60:
                rc = lib.exp_flux_cpa(lanes - 60, *common[1:], sms, stream)
            elif lanes >= 40:
                rc = lib.exp_flux_own(lanes - 40, *common[1:], sms, stream)
            elif lanes >= 30:
                rc = lib.exp_flux_aos(5 if lanes == 31 else 2, *common[1:], sms, stream)
            elif lanes >= 20:
                rc = lib.exp_flux_split(lanes - 20, *common[1:], sms, stream)
            elif lanes >= 10:
                rc = lib.exp_flux_h(lanes - 10, *common[1:], sms * 2, stream)
            elif lanes >= 6:
                rc = lib.exp_flux_reg(lay + 2 * (lanes - 5), *common[1:], sms, stream)
            elif lanes >= 3:
                kk = {3: 3, 4: 2, 5: 4}[lanes]
                rc = lib.exp_flux_lock(lay + 2 * kk, *common[1:], sms * 2, stream)
            elif lanes == 2:
                rc = lib.exp_flux_lrec(lay, T["w"].data_ptr(), T["q"].data_ptr(), T["x"].data_ptr(),
                                       T["lim"].data_ptr(), T["grad"].data_ptr(), T["aux"].data_ptr(),
                                       T["res"].data_ptr(), slots.data_ptr(), n, ints["lrec"].data_ptr(),
                                       ints["tmask"].data_ptr(), ntask, sms * 2, stream)
            elif lanes:
                rc = lib.exp_flux_lanes(*common, ints["wrow"].data_ptr(), int(wrow.size - 1), sms * 2, stream)
            else:
                rc = lib.exp_flux_run(*common, sms, stream) if lay >= 2 else lib.exp_flux_run(*common, sms * 2, stream)
            assert rc == 0, rc
        launch()
        torch.cuda.synchronize()
        r = T["res"].cpu().numpy()
        if lay == 4:
            rr = r.reshape(n, 6)
        else:
            rr = r.reshape(6, n).T if lay % 2 == 0 else from_aosoa(r, n, 6)
        results[name] = rr, slots.cpu().numpy()
        T["res"].copy_(res0)
        for _ in range(5):
            launch()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize()
        a.record()
        for _ in range(args.reps):
            launch()
        b.record()
        b.synchronize()
        out[name] = a.elapsed_time(b) / args.reps
    same = {k: all(np.array_equal(results["soa"][i], results[k][i]) for i in range(2)) for k in results}
    print(json.dumps({"grid": args.grid, "edges": m, "warp_tasks": int(wrow.size - 1),
                      "lane_util": float(m / (32 * (wrow.size - 1))), "ms": out, "bitwise_equal_to_soa": same}))


if __name__ == "__main__":
    main()
