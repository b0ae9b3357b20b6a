"""Summarise ncu captures for profiles/ (run in the build container).

    python scripts/ncu_summary.py gpurun_out/r05/edge_loops.ncu-rep --b-alg vflux=464278784 ... \
        --out profiles/r1_edge_loops.md [--launches gpurun_out/r05/launches.csv]

Per kernel: duration, DRAM bytes read/written (traffic), DRAM throughput %,
L1/L2 hit rates, registers, occupancy limits and the main stall reasons; with
--b-alg, the algorithmic bytes, achieved GB/s and traffic / B_alg.
"""
from __future__ import annotations

import argparse
import collections
import csv
import io
import json
import re
import subprocess
import sys

METRICS = [
    ("gpu__time_duration.sum", "duration"),
    ("dram__bytes_read.sum", "dram_read"),
    ("dram__bytes_write.sum", "dram_write"),
    ("gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "dram_pct"),
    ("lts__t_sector_hit_rate.pct", "l2_hit_pct"),
    ("l1tex__t_sector_hit_rate.pct", "l1_hit_pct"),
    ("launch__registers_per_thread", "regs"),
    ("launch__grid_size", "grid"),
    ("launch__block_size", "block"),
    ("launch__shared_mem_per_block_dynamic", "dyn_smem"),
    ("sm__warps_active.avg.per_cycle_active", "warps_per_sm"),
    ("smsp__issue_active.avg.pct_of_peak_sustained_active", "issue_pct"),
    ("smsp__average_warps_issue_stalled_long_scoreboard_per_issue_active.ratio", "stall_long_sb"),
    ("smsp__average_warps_issue_stalled_barrier_per_issue_active.ratio", "stall_barrier"),
    ("smsp__average_warps_issue_stalled_wait_per_issue_active.ratio", "stall_wait"),
]
UNIT = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "nsecond": 1e-9, "usecond": 1e-6,
        "msecond": 1e-3, "second": 1, "ns": 1e-9, "us": 1e-6, "ms": 1e-3, "s": 1,
        "B": 1, "KB": 1e3, "MB": 1e6, "GB": 1e9}


def read_raw(rep: str):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True,
                         text=True, check=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr, units = rows[0], rows[1]
    for r in rows[2:]:
        rec = {"kernel": r[hdr.index("Kernel Name")]}
        for m, key in METRICS:
            if m in hdr:
                i = hdr.index(m)
                v = float(r[i].replace(",", "")) if r[i] else float("nan")
                rec[key] = v * UNIT.get(units[i], 1)
        yield rec


def short(name: str) -> str:
    m = re.search(r"(k_[a-z_0-9]+)<(?:.*?::)?(\w+), (double|long)", name)
    if m:
        return f"{m.group(1)}<{m.group(2)}>"
    m = re.search(r"(k_[a-z_0-9]+)", name)
    return m.group(1) if m else name[:60]


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("rep")
    ap.add_argument("--b-alg", nargs="*", default=[], help="Functor=bytes (algorithmic bytes per launch)")
    ap.add_argument("--out", required=True)
    ap.add_argument("--launches", default=None)
    ap.add_argument("--title", default="ncu summary")
    args = ap.parse_args()
    balg = {k: int(v) for k, v in (x.split("=") for x in args.b_alg)}
    lines = [f"# {args.title}", "", f"source: `{args.rep}` (ncu --set full, --clock-control none;"
             " per-launch, cold and serialised: compare shares, not absolutes)", "",
             "| kernel | µs | DRAM rd MB | DRAM wr MB | traffic/B_alg | B_alg GB/s | DRAM % | L2 hit % | "
             "L1 hit % | regs | warps/SM | issue % | stall long-sb | stall barrier |",
             "|---|---|---|---|---|---|---|---|---|---|---|---|---|---|"]
    traffic = {}
    for r in read_raw(args.rep):
        k = short(r["kernel"])
        functor = next((f for f in balg if f.lower() in k.lower()), None)
        ba = balg.get(functor)
        tr = r.get("dram_read", 0) + r.get("dram_write", 0)
        dur = r["duration"]
        ratio = f"{tr / ba:.2f}" if ba else "-"
        gbs = f"{ba / dur / 1e9:.0f}" if ba else "-"
        if functor:
            traffic[functor] = int(tr)
        lines.append(f"| {k} | {dur * 1e6:.1f} | {r.get('dram_read', 0) / 1e6:.1f} | "
                     f"{r.get('dram_write', 0) / 1e6:.1f} | {ratio} | {gbs} | {r.get('dram_pct', 0):.1f} | "
                     f"{r.get('l2_hit_pct', 0):.1f} | {r.get('l1_hit_pct', 0):.1f} | {r.get('regs', 0):.0f} | "
                     f"{r.get('warps_per_sm', 0):.1f} | {r.get('issue_pct', 0):.1f} | "
                     f"{r.get('stall_long_sb', 0):.2f} | {r.get('stall_barrier', 0):.2f} |")
    if args.launches:
        rows = list(csv.reader(open(args.launches)))
        hi = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
        hdr = rows[hi]
        ki, vi = hdr.index("Kernel Name"), hdr.index("Metric Value")
        agg = collections.OrderedDict()
        for r in rows[hi + 1:]:
            a = agg.setdefault(short(r[ki]), [0, 0.0])
            a[0] += 1
            a[1] += float(r[vi].replace(",", ""))
        tot = sum(v[1] for v in agg.values())
        lines += ["", f"## launch list (`{args.launches}`, gpu__time_duration.sum, ns)", "",
                  "| kernel | launches | total µs | share % |", "|---|---|---|---|"]
        for k, (n, t) in sorted(agg.items(), key=lambda x: -x[1][1]):
            lines.append(f"| {k} | {n} | {t / 1e3:.1f} | {100 * t / tot:.1f} |")
    open(args.out, "w").write("\n".join(lines) + "\n")
    print("\n".join(lines))
    if traffic:
        print(json.dumps(traffic))


if __name__ == "__main__":
    sys.exit(main())
