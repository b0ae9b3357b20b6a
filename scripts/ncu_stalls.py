"""Top stalled SASS instructions per kernel in an ncu report (source page)."""
import csv
import subprocess
import sys

rep, pat = sys.argv[1], (sys.argv[2] if len(sys.argv) > 2 else "")
ntop = int(sys.argv[3]) if len(sys.argv) > 3 else 14
data = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv"], capture_output=True,
                      text=True).stdout
seen = set()
for b in data.split('"Kernel Name",')[1:]:
    lines = b.splitlines()
    name = lines[0]
    if pat not in name or name in seen:
        continue
    seen.add(name)
    rows = list(csv.reader(lines[1:]))
    hdr = rows[0]
    si = hdr.index("Warp Stall Sampling (All Samples)")
    recs, tot = [], 0.0
    for i, r in enumerate(rows[1:]):
        if len(r) < len(hdr):
            continue
        v = float(r[si])
        tot += v
        recs.append((v, i, r[1].strip()))
    print("=====", name[:100], "samples", int(tot))
    for v, i, s in sorted(recs, reverse=True)[:ntop]:
        ctx = " | ".join(x[2][:40] for x in recs[max(0, i - 2):i])
        print(f"  {100 * v / tot:5.1f}% #{i}: {s[:60]:60s}  <- {ctx}")
