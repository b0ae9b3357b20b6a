#!/usr/bin/env bash
# One measurement pass: bench line (no CPU leg), ncu launch list of the same
# command, one `ncu --set full` capture of every kernel of one iteration.
# Usage: gpurun -- bash scripts/gpu_round.sh <tag>
set -u
TAG=${1:-round}
OUT=gpurun_out/$TAG; mkdir -p "$OUT"
timeout 900 python bench.py --steps 20 --warmup 5 --no-cpu --scale-grid 0 > "$OUT/bench.json" 2> "$OUT/bench.err"
echo "bench rc=$?" >> "$OUT/status.txt"
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file "$OUT/launches.csv" \
  python bench.py --steps 2 --warmup 1 --no-cpu --scale-grid 0 > "$OUT/launches.log" 2>&1
echo "launches rc=$?" >> "$OUT/status.txt"
timeout 1200 ncu --set full --clock-control none --import-source on --kernel-name-base demangled \
  -k "regex:k_pfold1|k_pfold_rest|k_gather|k_direct" -s 6 -c 6 -o "$OUT/iteration" \
  python scripts/profile_proxy.py --iters 2 --inc-schedule auto > "$OUT/ncu_full.log" 2>&1
echo "ncu full rc=$?" >> "$OUT/status.txt"
cat "$OUT/status.txt"
