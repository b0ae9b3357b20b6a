#!/usr/bin/env bash
# Segmented-SOA parameter sweep: rebuild with each (shift, pad), bench once.
# Usage: gpurun -- bash scripts/seg_sweep.sh <tag> "12:32 5:0 12:32:8 ..." (shift:pad[:max dim])
set -u
TAG=${1:-segsweep}; VARIANTS=${2:-"12:32 5:0 8:0 10:32 12:512"}
OUT=gpurun_out/$TAG; mkdir -p "$OUT"
for v in $VARIANTS; do
  IFS=: read -r sh pad mx <<< "$v"; mx=${mx:-64}
  MESHLOOP_NVCC_FLAGS="-DML_SEG_SHIFT=$sh -DML_SEG_PAD=$pad -DML_SEG_MAX_DIM=$mx" python -c \
    "from paper_1403_7209_b200 import _build; _build.build(force=True)" > "$OUT/build_$v.log" 2>&1
  timeout 600 python bench.py --steps 20 --warmup 5 --no-cpu --scale-grid 0 --schedule-table "iflux+vflux=pfold" \
    > "$OUT/bench_$v.json" 2> "$OUT/bench_$v.err"
  python - "$OUT/bench_$v.json" "$v" <<'PY'
import json, sys
d = json.loads(open(sys.argv[1]).read().splitlines()[-1])
print(sys.argv[2], round(d["ms_per_step"], 4), {k: v["ms"] for k, v in d["loops"].items()})
PY
done
