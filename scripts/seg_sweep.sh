#!/usr/bin/env bash
# Segmented-SOA parameter sweep: rebuild with each (shift, pad), bench once.
# Usage: gpurun -- bash scripts/seg_sweep.sh <tag> "6:0 5:0:19:18 ..." (shift:pad[:max dim[:min dim]])
set -u
TAG=${1:-segsweep}; VARIANTS=${2:-"6:0 5:0 4:0 7:0 6:0:64:2"}
OUT=gpurun_out/$TAG; mkdir -p "$OUT"
for v in $VARIANTS; do
  IFS=: read -r sh pad mx mn <<< "$v"; mx=${mx:-64}; mn=${mn:-8}
  MESHLOOP_NVCC_FLAGS="-DML_SEG_SHIFT=$sh -DML_SEG_PAD=$pad -DML_SEG_MAX_DIM=$mx -DML_SEG_MIN_DIM=$mn" python -c \
    "from paper_1403_7209_b200 import _build; _build.build(force=True)" > "$OUT/build_$v.log" 2>&1
  timeout 600 python bench.py --steps 20 --warmup 5 --no-cpu --scale-grid 0 --schedule-table "iflux+vflux=pfold" \
    > "$OUT/bench_$v.json" 2> "$OUT/bench_$v.err"
  python - "$OUT/bench_$v.json" "$v" <<'PY'
import json, sys
d = json.loads(open(sys.argv[1]).read().splitlines()[-1])
print(sys.argv[2], round(d["ms_per_step"], 4), {k: v["ms"] for k, v in d["loops"].items()})
PY
done
