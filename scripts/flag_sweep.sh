#!/usr/bin/env bash
# Build-flag A/B sweep: rebuild with each flag set, bench once, print per-loop ms.
# Usage: gpurun -- bash scripts/flag_sweep.sh <tag> "label=-DFOO=1 -DBAR=2|label2=..." [bench args]
set -u
TAG=${1:-flags}; VARIANTS=${2:-"default="}; shift 2 || true
OUT=gpurun_out/$TAG; mkdir -p "$OUT"
IFS='|' read -ra VS <<< "$VARIANTS"
for v in "${VS[@]}"; do
  label=${v%%=*}; flags=${v#*=}
  MESHLOOP_NVCC_FLAGS="$flags" python -c \
    "from paper_1403_7209_b200 import _build; _build.build(force=True)" > "$OUT/build_$label.log" 2>&1
  timeout 600 python bench.py --steps 20 --warmup 5 --no-cpu --scale-grid 0 "$@" \
    > "$OUT/bench_$label.json" 2> "$OUT/bench_$label.err"
  python - "$OUT/bench_$label.json" "$label" <<'PY'
import json, sys
d = json.loads(open(sys.argv[1]).read().splitlines()[-1])
print(sys.argv[2], round(d["ms_per_step"], 4), {k: v["ms"] for k, v in d["loops"].items()})
PY
done
