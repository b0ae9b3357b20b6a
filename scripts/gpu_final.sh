#!/usr/bin/env bash
# Round-end evidence pass: GPU tests, smoke(), bench lines (device-only and
# default with the CPU leg), the reference arm, the ncu launch list of the
# bench command (cold, the recipe's pass), a warm launch list of an eager
# iteration (--cache-control none: kernel-time sum vs the graph iteration),
# and one `ncu --set full` capture of every kernel of one iteration.
# Usage: gpurun -- bash scripts/gpu_final.sh <tag>
set -u
TAG=${1:-final}
OUT=gpurun_out/$TAG; mkdir -p "$OUT"; : > "$OUT/status.txt"
timeout 1500 python -m pytest tests -m gpu -x -q > "$OUT/pytest_gpu.log" 2>&1
echo "pytest rc=$? $(tail -1 "$OUT/pytest_gpu.log")" >> "$OUT/status.txt"
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > "$OUT/smoke.log" 2>&1
echo "smoke rc=$?" >> "$OUT/status.txt"
bash scripts/gpu_round.sh "$TAG" > /dev/null 2>&1
cat "$OUT/status.txt" > /dev/null
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --cache-control none -c 400 --csv \
  --log-file "$OUT/launches_warm.csv" python scripts/profile_proxy.py --iters 4 --inc-schedule auto \
  > "$OUT/launches_warm.log" 2>&1
echo "warm launches rc=$?" >> "$OUT/status.txt"
timeout 900 python bench.py > "$OUT/bench_default.json" 2> "$OUT/bench_default.err"
echo "default bench rc=$?" >> "$OUT/status.txt"
timeout 900 python bench.py --impl reference > "$OUT/bench_ref.json" 2> "$OUT/bench_ref.err"
echo "reference rc=$?" >> "$OUT/status.txt"
cat "$OUT/status.txt"
