#!/usr/bin/env bash
# compute-sanitizer over every kernel family (scripts/sanitize_cases.py):
# memcheck, racecheck, synccheck and initcheck on one GPU, then memcheck on
# the 2-rank owner-compute path (NVLink IPC halos + reductions, ranks sharing
# the GPU).  Summaries go to gpurun_out/<tag>/sanitize_*.log.
set -u
TAG=${1:-sanitize}
OUT=gpurun_out/$TAG; mkdir -p "$OUT"
CS="compute-sanitizer --print-limit 50 --error-exitcode 9"
for tool in memcheck racecheck synccheck initcheck; do
  timeout 1200 $CS --tool $tool python scripts/sanitize_cases.py > "$OUT/sanitize_$tool.log" 2>&1
  echo "$tool rc=$?" >> "$OUT/status.txt"
done
timeout 1200 $CS --tool memcheck --target-processes all python scripts/sanitize_cases.py --ranks 2 \
  > "$OUT/sanitize_ranks_memcheck.log" 2>&1
echo "ranks memcheck rc=$?" >> "$OUT/status.txt"
timeout 1200 $CS --tool synccheck --target-processes all python scripts/sanitize_cases.py --ranks 2 \
  > "$OUT/sanitize_ranks_synccheck.log" 2>&1
echo "ranks synccheck rc=$?" >> "$OUT/status.txt"
cat "$OUT/status.txt"
