"""Device residency: HBM mirrors of dats, maps and plans.

Layout in HBM:

* a dat is one float64/int64 buffer, uploaded on first use and kept
  resident across ``run_program`` calls: AOS ``e*dim+c`` as on the host; SOA
  (dim > 1) *segmented* — 4096-element segments each storing its components
  one after another (``SEG_SHIFT``), copied to/from the host's ``c*size+e``
  with one 2-D transfer of 32 KB rows plus a tail per component;
* a map is stored int32 and column-major (``[arity][from_size]``), so the
  index reads of one map column by consecutive elements are coalesced and
  cost 4 B per element instead of the host table's 8 B;
* a plan is three arrays: block ids ordered by colour (int32), element
  colours (uint16) and per-block colour counts (int32).

Coherence is lazy and conservative: ``Dat.data`` (which may be written
through) marks the mirror host-newer; executions mark written dats
device-newer and the host copy is refreshed on the next host access.
"""
from __future__ import annotations

import numpy as np

from . import _native as N
from .core import AOS, Dat, ExecError, Map

__all__ = ["DatMirror", "dat_mirror", "segmented", "device_elems", "device_pitch", "PITCH_ALIGN", "map_mirror", "plan_mirror", "pin_mesh",
           "gather_mirror", "pfold_mirror", "gather_eligible", "fold_eligible", "SEG_SHIFT"]


#: SOA dats of dim > 1 are stored *segmented* on the device: segments of
#: S = 2**SEG_SHIFT elements, each holding its components one after another
#: at stride P = S + SEG_PAD — (e, c) at (e >> s) * P * dim + c * P + (e % S).
#: Inside a segment a component is a contiguous run (coalesced like plain
#: SOA); the offset of component c from an element's base is the
#: compile-time c * P * 8 bytes, a load immediate in the kernels (engine.cuh).
def _seg_params():
    global SEG_SHIFT, SEG_PAD, SEG_MAX_DIM, SEG_MIN_DIM
    if SEG_SHIFT is None:
        SEG_SHIFT, SEG_PAD, SEG_MAX_DIM, SEG_MIN_DIM = N.seg_params()   # as the library was built
    return SEG_SHIFT, SEG_PAD


#: segment shift / component pad / widest and narrowest segmented dim, read from the library
SEG_SHIFT = SEG_PAD = SEG_MAX_DIM = SEG_MIN_DIM = None


def segmented(dat: Dat) -> bool:
    """Whether ``dat``'s device copy is segmented SOA (SOA, dim within the
    library's segmented range and > 1); other SOA dats keep plain rows."""
    _seg_params()
    return dat.layout is not AOS and 1 < dat.dim and SEG_MIN_DIM <= dat.dim <= SEG_MAX_DIM


#: plain SOA rows (dims above the segmented range) are padded to this many
#: elements, so every component row starts 256-byte aligned and the pitch is
#: even (16-byte element pairs in the direct loops)
PITCH_ALIGN = 32


def device_pitch(dat: Dat) -> int:
    """Component stride of a plain (unsegmented) device copy: the set size, or
    for SOA dats of dim > 1 the set size rounded up to PITCH_ALIGN."""
    n = dat.set.size
    if dat.layout is AOS or dat.dim == 1:
        return n
    return -(-n // PITCH_ALIGN) * PITCH_ALIGN


def device_elems(dat: Dat) -> int:
    """Elements of ``dat``'s device copy (segmented copies round the set up to
    whole segments, pitched ones pad each component row)."""
    n = dat.set.size
    if not segmented(dat):
        return device_pitch(dat) * dat.dim
    sh, pad = _seg_params()
    seg = 1 << sh
    return -(-n // seg) * (seg + pad) * dat.dim


class DatMirror:
    """Device copy of one dat payload: AOS rows (and dim-1 dats) as on the
    host; SOA dats segmented (``SEG_SHIFT``), copied with one 2-D transfer of
    the full segments plus one tail copy per component (``ml_seg_copy``)."""

    __slots__ = ("buf", "layout", "nbytes", "host_newer", "device_newer", "seg", "n", "dim", "isz",
                 "_pitch")

    def __init__(self):
        self.buf = None
        self.layout = None
        self.nbytes = -1
        self.host_newer = True
        self.device_newer = False
        self.seg = False
        self.n = self.dim = self.isz = self._pitch = 0

    @property
    def ptr(self) -> int:
        return self.buf.ptr if self.buf is not None else 0

    @property
    def pitch(self) -> int:
        """ABI ``pitch`` of the copy (plain SOA component stride)."""
        return self._pitch

    @property
    def padded(self) -> bool:
        return not self.seg and self._pitch != self.n and self.dim > 1

    @property
    def seg_shift(self) -> int:
        return _seg_params()[0] if self.seg else 0

    def strides(self, dat: Dat) -> tuple[int, int]:
        """(element stride, component stride) in the ABI's row-kernel
        convention (ml_pack_rows): a negative element stride -S = segmented
        SOA with segments of S elements."""
        if self.seg:
            sh, pad = _seg_params()
            return -(1 << sh), (1 << sh) + pad
        return (dat.dim, 1) if dat.layout is AOS else (1, self._pitch)

    def _seg_copy(self, host: np.ndarray, to_device: bool, stream: int) -> None:
        N.check(N.lib().ml_seg_copy(self.buf.ptr, N.ptr(host), self.n, self.dim, self.isz, _seg_params()[0],
                                    int(to_device), stream), "ml_seg_copy")

    def upload(self, host: np.ndarray) -> None:
        if self.buf is None or not host.nbytes:
            return
        if self.seg:
            self._seg_copy(host, True, N.ML_STREAM_COMPUTE)
        elif self.padded:
            rb = self.n * self.isz
            N.check(N.lib().ml_upload2d(self.buf.ptr, self._pitch * self.isz, N.ptr(host), rb, rb, self.dim),
                    "ml_upload2d")
        else:
            self.buf.upload(host)

    def download(self, host: np.ndarray) -> None:
        if self.buf is not None and host.nbytes:
            if not host.flags.c_contiguous:
                raise ExecError("dat payload must be contiguous to receive device data")
            if self.seg:
                self._seg_copy(host, False, N.ML_STREAM_COMPUTE)
            elif self.padded:
                rb = self.n * self.isz
                N.check(N.lib().ml_download2d(N.ptr(host), rb, self.buf.ptr, self._pitch * self.isz, rb,
                                              self.dim), "ml_download2d")
            else:
                self.buf.download(host)
        self.device_newer = False

    def copy_h2d(self, host: np.ndarray) -> None:
        """Asynchronous upload on the H2D copy stream (streamed residency)."""
        if self.buf is None or not host.nbytes:
            return
        if self.seg:
            self._seg_copy(host, True, N.ML_STREAM_H2D)
        elif self.padded:
            rb = self.n * self.isz
            N.check(N.lib().ml_copy_h2d_2d(self.buf.ptr, self._pitch * self.isz, N.ptr(host), rb, rb,
                                           self.dim), "ml_copy_h2d_2d")
        else:
            N.check(N.lib().ml_copy_h2d(self.buf.ptr, N.ptr(host), host.nbytes), "ml_copy_h2d")

    def copy_d2h(self, host: np.ndarray) -> None:
        """Asynchronous download on the D2H copy stream (streamed residency)."""
        if self.buf is None or not host.nbytes:
            return
        if self.seg:
            self._seg_copy(host, False, N.ML_STREAM_D2H)
        elif self.padded:
            rb = self.n * self.isz
            N.check(N.lib().ml_copy_d2h_2d(N.ptr(host), rb, self.buf.ptr, self._pitch * self.isz, rb,
                                           self.dim), "ml_copy_d2h_2d")
        else:
            N.check(N.lib().ml_copy_d2h(N.ptr(host), self.buf.ptr, host.nbytes), "ml_copy_d2h")


def dat_mirror(dat: Dat, force_upload: bool = False, upload: bool = True) -> DatMirror:
    """The up-to-date device mirror of ``dat`` (allocating/uploading as needed;
    ``upload=False`` only allocates — the caller copies the contents)."""
    m = dat._dev
    if m is None:
        m = dat._dev = DatMirror()
    host = dat._host
    seg = segmented(dat)
    dev_bytes = device_elems(dat) * host.dtype.itemsize if host.nbytes else 0
    if m.buf is None or m.nbytes != dev_bytes or m.seg != seg:
        if m.device_newer:
            raise ExecError(f"dat {dat.name!r}: payload resized while device data is newer")
        m.buf = N.DeviceBuffer(dev_bytes) if dev_bytes else None
        m.nbytes = dev_bytes
        m.host_newer = True
    m.seg, m.n, m.dim, m.isz = seg, dat.set.size, dat.dim, host.dtype.itemsize
    m._pitch = device_pitch(dat)
    if m.layout is not dat.layout:
        m.layout = dat.layout
        m.host_newer = True
    if upload and (m.host_newer or force_upload) and not m.device_newer:
        if host.nbytes:
            if not host.flags.c_contiguous:
                dat._host = host = np.ascontiguousarray(host)
            m.upload(host)
        m.host_newer = False
    return m


class _MapMirror:
    __slots__ = ("buf", "table", "shape")

    def __init__(self, buf, table):
        self.buf = buf
        self.table = table
        self.shape = table.shape


def map_mirror(m: Map) -> int:
    """Device pointer of the int32 column-major copy of ``m.table``."""
    mm = m._dev
    if mm is not None and mm.table is m.table and mm.shape == m.table.shape:
        return mm.buf.ptr if mm.buf is not None else 0
    t = np.ascontiguousarray(m.table, dtype=np.int64)
    if t.size and int(t.max(initial=0)) >= 2 ** 31:
        raise ExecError(f"map {m.name!r}: ids exceed int32")
    buf = N.DeviceBuffer(t.size * 4) if t.size else None
    if t.size:
        N.check(N.lib().ml_map_upload(buf.ptr, N.ptr(t), t.shape[0], t.shape[1]), "ml_map_upload")
    m._dev = _MapMirror(buf, m.table)
    return buf.ptr if buf is not None else 0


class PlanMirror:
    __slots__ = ("blocks", "ecol", "encol", "offsets")

    def __init__(self, plan):
        blocks = plan.blocks_flat.astype(np.int32)
        self.offsets = np.ascontiguousarray(plan.color_offsets, dtype=np.int64)
        self.blocks = N.DeviceBuffer(max(blocks.nbytes, 4))
        if blocks.size:
            self.blocks.upload(blocks)
        self.ecol = self.encol = None
        if plan.has_writes:
            if plan.max_elem_colors > 65535:
                raise ExecError("more than 65535 element colours in one block")
            ecol = plan.elem_color.astype(np.uint16)
            encol = plan.elem_ncolors.astype(np.int32)
            self.ecol = N.DeviceBuffer(max(ecol.nbytes, 4))
            self.encol = N.DeviceBuffer(max(encol.nbytes, 4))
            if ecol.size:
                self.ecol.upload(ecol)
                self.encol.upload(encol)


def plan_mirror(plan) -> PlanMirror:
    if plan._dev is None:
        plan._dev = PlanMirror(plan)
    return plan._dev


#: incidences per gather row before a target is split across rows (hub targets)
HUB_ROW = 128


def gather_lists_host(loop, n: int, hubs: bool = False, hub_row: int = HUB_ROW) -> dict:
    """Host arrays of the gather schedule (ml_gather_build): per target row its
    (element, written-argument position) incidences in serial order.  Rows are
    compacted to touched targets when fewer than half are touched
    (``targets``: row -> target id, else None = identity).  With ``hubs`` (INC
    only) a target with more than ``hub_row`` incidences is split into rows of
    at most ``hub_row``: ``seg[row]`` is the row's partial slot (-1: ordinary
    row), ``hub_tl``/``hub_off`` list each hub target and its slots.
    ``host`` keeps the one-row-per-target lists (pfold, multi-GPU subsets)."""
    import ctypes as C
    wr = [a for a in loop.args if a.kind == "indirect" and a.mode.name != "READ"]
    nset = wr[0].dat.set.size
    cols = [np.ascontiguousarray(a.map.table[:n, a.slot], dtype=np.int64) for a in wr]
    L = N.lib()
    h = C.c_void_p()
    cptr = (C.c_void_p * len(cols))(*[N.ptr(c) for c in cols])
    N.check(L.ml_gather_build(n, len(cols), cptr, nset, C.byref(h)), "ml_gather_build")
    try:
        off = np.empty(nset + 1, np.int32)
        elem = np.empty(max(n * len(cols), 1), np.int32)
        pos = np.empty(max(n * len(cols), 1), np.uint8)
        N.check(L.ml_gather_export(h, N.ptr(off), N.ptr(elem), N.ptr(pos)), "ml_gather_export")
    finally:
        L.ml_gather_free(h)
    deg = np.diff(off)
    touched = np.flatnonzero(deg)
    tl = None
    if 2 * touched.size < nset:
        off = np.concatenate([[0], np.cumsum(deg[touched])]).astype(np.int32)
        tl = touched.astype(np.int32)
    out = {"host": {"off": off, "elem": elem, "pos": pos,
                    "targets": tl if tl is not None else np.arange(off.size - 1, dtype=np.int32)},
           "elem": elem, "pos": pos, "seg": None, "nhub": 0, "nslots": 0,
           "hub_tl": None, "hub_off": None}
    if hubs and wr[0].mode.name == "INC":
        sp = split_hub_rows(off, tl if tl is not None else np.arange(off.size - 1, dtype=np.int32),
                            hub_row)
        if sp is not None:
            off, tl = sp["off"], sp["targets"]
            out.update({k: sp[k] for k in ("seg", "nhub", "nslots", "hub_tl", "hub_off")})
    out["off"], out["targets"] = off, tl
    return out


def split_hub_rows(off: np.ndarray, rows_tl: np.ndarray, hub_row: int = HUB_ROW):
    """Split every row of a CSR with more than ``hub_row`` entries into rows of
    at most ``hub_row`` (same entry order).  Returns None when no row is that
    long, else the new ``off``/``targets`` and, per new row, its partial slot
    ``seg`` (-1: ordinary row); ``hub_tl``/``hub_off``: each split target and
    its partial slots, in row (= element) order."""
    deg = np.diff(off)
    heavy = np.flatnonzero(deg > hub_row)
    if not heavy.size:
        return None
    nseg = np.where(deg > hub_row, -(-deg // hub_row), 1)
    row_target = np.repeat(np.arange(deg.size), nseg)
    first = np.concatenate([[0], np.cumsum(nseg)])[:-1]
    within = np.arange(row_target.size) - np.repeat(first, nseg)
    row_lo = off[row_target] + within * hub_row
    row_hi = np.minimum(row_lo + hub_row, off[row_target + 1])
    is_hub_row = deg[row_target] > hub_row
    seg = np.full(row_target.size, -1, np.int32)
    seg[is_hub_row] = np.arange(int(is_hub_row.sum()), dtype=np.int32)
    return {"off": np.concatenate([row_lo, row_hi[-1:]]).astype(np.int32),
            "targets": rows_tl[row_target].astype(np.int32), "seg": seg,
            "nhub": int(heavy.size), "nslots": int(is_hub_row.sum()),
            "hub_tl": rows_tl[heavy].astype(np.int32),
            "hub_off": np.concatenate([[0], np.cumsum(nseg[heavy])]).astype(np.int32)}


def pfold_lists_host(host: dict, hub_row: int | None = HUB_ROW) -> dict:
    """Primary-fold lists from one-row-per-target gather lists.

    Each element's *primary* incidence is its first INC argument: the owner
    of that target evaluates the element and keeps that increment; the other
    incidences are *secondary* (slots).  Per
    target: its primary incidences (``1``) and its secondary ones (``2``,
    with their argument positions ``pos2``), element
    ascending; only targets that have any.  Rows longer than ``hub_row`` are
    split (``split_hub_rows``): ``seg{1,2}``, ``nhub{1,2}``, ``nslots{1,2}``,
    ``hub{1,2}_tl``, ``hub{1,2}_off``."""
    off, elem, pos, tl = host["off"], host["elem"], host["pos"], host["targets"]
    nt = off.size - 1
    owner = np.repeat(np.arange(nt), np.diff(off))
    e, p_ = elem[:off[-1]], pos[:off[-1]]
    # primary = the first INC argument: after the reference's row ordering of
    # the iteration set (renumber.py:131-138) an element's edge ids follow its
    # first target, so a target's primary elements are consecutive ids and
    # their direct rows and records stream coalesced (a smallest-target rule
    # measured 2 % slower on the fused flux loop)
    prim = p_ == 0
    out = {}
    for which in (1, 2):
        m = prim if which == 1 else ~prim
        cnt = np.bincount(owner[m], minlength=nt)
        keep = np.flatnonzero(cnt)
        out[f"n{which}"] = int(keep.size)
        out[f"off{which}"] = np.concatenate([[0], np.cumsum(cnt[keep])]).astype(np.int32)
        out[f"elem{which}"] = np.ascontiguousarray(e[m], dtype=np.int32)
        out[f"tl{which}"] = np.ascontiguousarray(tl[keep], dtype=np.int32)
        out["ppos1" if which == 1 else "pos2"] = np.ascontiguousarray(p_[m], dtype=np.uint8)
    # slot row of each (element, secondary position): its index in the secondary
    # CSR; an element's secondary positions are numbered in ascending order
    # skipping its primary position
    nw = int(p_.max(initial=0)) + 1 if p_.size else 1
    n_el = int(e.max(initial=-1)) + 1
    slotpos = np.zeros(max(n_el * max(nw - 1, 1), 1), np.int32)
    if nw > 1 and out["elem2"].size:
        pp = np.zeros(max(n_el, 1), np.int64)
        pp[out["elem1"]] = out["ppos1"]
        e2, p2 = out["elem2"].astype(np.int64), out["pos2"].astype(np.int64)
        j = p2 - (p2 > pp[e2])
        slotpos[e2 * (nw - 1) + j] = np.arange(e2.size, dtype=np.int32)
    out["slotpos"] = slotpos
    for which in (1, 2):
        sp = split_hub_rows(out[f"off{which}"], out[f"tl{which}"], hub_row) if hub_row else None
        if sp is None:
            out.update({f"seg{which}": None, f"nhub{which}": 0, f"nslots{which}": 0,
                        f"hub{which}_tl": None, f"hub{which}_off": None})
            continue
        out[f"off{which}"], out[f"tl{which}"] = sp["off"], sp["targets"]
        out[f"n{which}"] = int(sp["off"].size - 1)
        out.update({f"seg{which}": sp["seg"], f"nhub{which}": sp["nhub"], f"nslots{which}": sp["nslots"],
                    f"hub{which}_tl": sp["hub_tl"], f"hub{which}_off": sp["hub_off"]})
    return out


class GatherMirror:
    """Device target-centric incidence lists (ml_gather_build) of a loop whose
    indirect writes are all INC, or all WRITE, of one dat.  When fewer than
    half of the target set's elements have incidences (e.g. boundary loops),
    the list is compacted to those targets (``targets``)."""

    __slots__ = ("off", "elem", "pos", "ntargets", "targets", "host", "seg", "part", "nhub",
                 "hub_tl", "hub_off", "rec", "ncol", "rcol", "rec_host")

    def __init__(self, loop, n: int, hubs: bool = False):
        wr = [a for a in loop.args if a.kind == "indirect" and a.mode.name != "READ"]
        h = gather_lists_host(loop, n, hubs)
        self.host = h["host"]
        # per-incidence map records: the kernel reads each incidence's map
        # entries beside its element id instead of through it
        self.rec_host, self.rcol = pfold_records_host(loop, h["elem"])
        self.ncol = self.rec_host.shape[1]
        self.rec = _upload(self.rec_host)
        self.seg = self.part = self.hub_tl = self.hub_off = None
        self.nhub = h["nhub"]
        if h["seg"] is not None:
            self.seg = _upload(h["seg"])
            self.part = N.DeviceBuffer(max(h["nslots"] * wr[0].dat.dim * 8, 8))
            self.hub_tl = _upload(h["hub_tl"])
            self.hub_off = _upload(h["hub_off"])
        self.targets = _upload(h["targets"]) if h["targets"] is not None else None
        self.ntargets = int(h["off"].size - 1)
        self.off, self.elem, self.pos = _upload(h["off"]), _upload(h["elem"]), _upload(h["pos"])

    def subset(self, targets_idx: np.ndarray) -> dict:
        """Device lists of a subset of this list's targets (positions into it, ascending)."""
        h = self.host
        off = h["off"]
        deg = (off[targets_idx + 1] - off[targets_idx]).astype(np.int64)
        starts = off[targets_idx].astype(np.int64)
        new_off = np.concatenate([[0], np.cumsum(deg)]).astype(np.int32)
        take = (np.repeat(starts - new_off[:-1], deg) + np.arange(int(deg.sum()))).astype(np.int64)
        return {"ntargets": int(targets_idx.size), "off": _upload(new_off),
                "rec": _upload(np.ascontiguousarray(self.rec_host[take])),
                "elem": _upload(np.ascontiguousarray(h["elem"][take])),
                "pos": _upload(np.ascontiguousarray(h["pos"][take])),
                "targets": _upload(np.ascontiguousarray(h["targets"][targets_idx], dtype=np.int32)),
                "elem_host": h["elem"][take]}


class PFoldMirror:
    """Device lists of the primary-fold schedule (see PFoldParams in
    csrc/engine.cuh), split from a loop's gather lists: per target, its
    incidences through the first INC argument (pass 1) and through the others
    (pass 2), element ascending; plus the per-element slot buffer."""

    __slots__ = ("n1", "off1", "elem1", "tl1", "n2", "off2", "elem2", "tl2", "pos2", "slotpos",
                 "rec", "ncol", "rcol", "seg1", "seg2", "nhub1", "nhub2", "hub1_tl", "hub1_off",
                 "hub2_tl", "hub2_off", "part1", "part2", "host", "rec_host")

    def __init__(self, g: GatherMirror, loop):
        h = pfold_lists_host(g.host)
        self.host, self.rec_host = h, None
        self.n1, self.n2 = h["n1"], h["n2"]
        for k in ("off1", "elem1", "tl1", "off2", "elem2", "tl2", "pos2", "slotpos"):
            setattr(self, k, _upload(h[k]))
        inc = next(a for a in loop.args if a.kind == "indirect" and a.mode.name == "INC")
        row = inc.dat.dim * np.dtype(inc.dat.dtype).itemsize
        for w in (1, 2):
            seg = h[f"seg{w}"]
            setattr(self, f"nhub{w}", h[f"nhub{w}"])
            for k in ("seg", "hub_tl", "hub_off"):
                key = f"{k[:3]}{w}{k[3:]}" if k != "seg" else f"seg{w}"
                setattr(self, key, _upload(h[key]) if seg is not None else None)
            setattr(self, f"part{w}", N.DeviceBuffer(max(h[f"nslots{w}"] * row, 8)) if seg is not None else None)
        rec, self.rcol = pfold_records_host(loop, h["elem1"])      # pass 1 reads them (required)
        self.ncol = rec.shape[1]
        self.rec = _upload(rec)
        self.rec_host = rec

    def pass1_subset(self, rows: np.ndarray) -> dict:
        """Device pass-1 lists of a subset of the pass-1 rows (ascending
        positions): ``n1``, ``off1``, ``elem1``, ``tl1``, ``seg1``, ``rec``
        (multi-GPU core/boundary launches)."""
        h = self.host
        off = h["off1"]
        deg = (off[rows + 1] - off[rows]).astype(np.int64)
        new_off = np.concatenate([[0], np.cumsum(deg)]).astype(np.int32)
        take = (np.repeat(off[rows].astype(np.int64) - new_off[:-1], deg)
                + np.arange(int(deg.sum()))).astype(np.int64)
        out = {"n1": int(rows.size), "off1": _upload(new_off),
               "elem1": _upload(np.ascontiguousarray(h["elem1"][take])),
               "tl1": _upload(np.ascontiguousarray(h["tl1"][rows])),
               "seg1": _upload(np.ascontiguousarray(h["seg1"][rows])) if h["seg1"] is not None else None,
               "rec": (_upload(np.ascontiguousarray(self.rec_host[take]))
                       if self.rec_host is not None else None)}
        return out


def pfold_records_host(loop, elem1: np.ndarray):
    """Pass-1 element records: for each incidence k, the map entries of element
    elem1[k] for every distinct (map, column) the loop's indirect arguments
    use, [incidences][columns] int32; and each argument's record column (-1:
    not indirect)."""
    cols, rcol = [], [-1] * 16
    for i, a in enumerate(loop.args):
        if a.kind != "indirect":
            continue
        key = (id(a.map), a.slot)
        hit = [j for j, (m, c) in enumerate(cols) if (id(m), c) == key]
        if hit:
            rcol[i] = hit[0]
        else:
            rcol[i] = len(cols)
            cols.append((a.map, a.slot))
    e = elem1.astype(np.int64)
    rec = np.empty((e.size, max(len(cols), 1)), np.int32)
    for j, (m, c) in enumerate(cols):
        rec[:, j] = m.table[e, c]
    return rec, rcol


def pfold_mirror(loop, plan) -> PFoldMirror:
    cache = plan.__dict__.setdefault("_pfolds", {})
    key = loop.signature()
    if key not in cache:
        cache[key] = PFoldMirror(gather_mirror(loop, plan), loop)
    return cache[key]


def gather_eligible(loop) -> bool:
    """Target-centric execution applies when the loop's indirect writes all go to
    one dat with one mode — INC, or WRITE — no direct argument is written, and
    that dat is not accessed in any other way by the loop."""
    ind_w = [a for a in loop.args if a.kind == "indirect" and a.mode.name != "READ"]
    if not ind_w or len({a.mode.name for a in ind_w}) != 1:
        return False
    if ind_w[0].mode.name not in ("INC", "WRITE"):
        return False
    if len({a.dat.name for a in ind_w}) != 1:
        return False
    if any(a.kind == "direct" and a.mode.name != "READ" for a in loop.args):
        return False
    name, mode = ind_w[0].dat.name, ind_w[0].mode.name
    return not any(a.kind != "global" and a.dat.name == name and a.mode.name != mode
                   for a in loop.args)


def fold_eligible(loop) -> bool:
    """The fold schedule applies when the loop's indirect writes are all INCs of
    one dat that the loop accesses in no other way (direct writes are fine: each
    element is evaluated once)."""
    ind_w = [a for a in loop.args if a.kind == "indirect" and a.mode.name != "READ"]
    if not ind_w or any(a.mode.name != "INC" for a in ind_w):
        return False
    if len({a.dat.name for a in ind_w}) != 1:
        return False
    name = ind_w[0].dat.name
    return not any(a.kind != "global" and a.dat.name == name and a.mode.name != "INC"
                   for a in loop.args)


def gather_mirror(loop, plan, hubs: bool = False) -> GatherMirror:
    """Gather lists of ``loop``; ``hubs`` splits heavy targets into several
    rows (the gather kernel only — the fold kernels need one row per target)."""
    cache = plan.__dict__.setdefault("_gathers", {})
    key = (loop.signature(), hubs)
    if key not in cache:
        cache[key] = GatherMirror(loop, plan.n, hubs)
    return cache[key]


def _upload(host: np.ndarray):
    buf = N.DeviceBuffer(max(host.nbytes, 4))
    if host.nbytes:
        buf.upload(host)
    return buf


_PINNED_KEEPALIVE: dict = {}


def pin_mesh(mesh, min_bytes: int = 1 << 20, device: int = 0) -> int:
    """Re-home every dat payload of at least ``min_bytes`` into pinned host memory
    (so host<->device copies run at full PCIe speed); returns the bytes pinned.
    Initialises the library on ``device`` if nothing has yet."""
    if not N._inited:                    # pinned allocations go through the library
        N.init(device)
    total = 0
    for d in mesh.dats.values():
        host = d._pull()
        if host.nbytes < min_bytes:
            continue
        pa = N.PinnedArray(host.shape, host.dtype)
        pa.array[...] = host
        _PINNED_KEEPALIVE[id(pa.array)] = pa
        d._host = pa.array
        total += host.nbytes
    return total
