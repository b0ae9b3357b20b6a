#!/usr/bin/env bash
# Gather-schedule occupancy / layout sweep + tests + a bench line.
set -u
TAG=${1:-occ}
OUT=gpurun_out/$TAG; mkdir -p "$OUT"
python -c "import __graft_entry__ as g; g.build()" > "$OUT/build.log" 2>&1
timeout 900 python -m pytest tests -q -m gpu -p no:cacheprovider -x > "$OUT/pytest_gpu.log" 2>&1; echo "pytest rc=$?" >> "$OUT/status.txt"
for m in 0 2 3 4; do
  for soa in 4 -1; do
    echo "== MINB=$m soa=$soa" >> "$OUT/sweep.log"
    ML_GATHER_MINB=$m timeout 300 python scripts/profile_proxy.py --iters 3 --soa $soa --inc-schedule gather >> "$OUT/sweep.log" 2>&1
  done
done
echo "sweep done" >> "$OUT/status.txt"
timeout 600 python bench.py > "$OUT/bench.json" 2> "$OUT/bench.err"; echo "bench rc=$?" >> "$OUT/status.txt"
cat "$OUT/status.txt"; tail -2 "$OUT/pytest_gpu.log"; grep -v "^$" "$OUT/sweep.log"
