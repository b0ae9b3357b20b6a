#!/usr/bin/env bash
# One gpurun call: smoke, GPU tests, bench, ncu launch list + full capture of the edge loops.
# Usage (from the build container):
#   /usr/local/graft/bin/gpurun --timeout 2400 -- bash scripts/gpu_check.sh [tag]
set -u
TAG=${1:-r01}
OUT=gpurun_out/$TAG
mkdir -p "$OUT"
nvidia-smi > "$OUT/nvidia-smi.txt" 2>&1
python -c "import __graft_entry__ as g; g.build()" > "$OUT/build.log" 2>&1
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > "$OUT/smoke.log" 2>&1; echo "smoke rc=$?" >> "$OUT/status.txt"
timeout 1500 python -m pytest tests -q -m gpu -p no:cacheprovider --durations=15 > "$OUT/pytest_gpu.log" 2>&1; echo "pytest rc=$?" >> "$OUT/status.txt"
timeout 300 python scripts/profile_proxy.py --iters 3 --inc-schedule gather pfold colour > "$OUT/schedules.log" 2>&1; echo "sched rc=$?" >> "$OUT/status.txt"
timeout 600 python bench.py --steps 20 --warmup 3 > "$OUT/bench.json" 2> "$OUT/bench.err"; echo "bench rc=$?" >> "$OUT/status.txt"
timeout 300 python bench.py --impl reference --steps 2 --warmup 1 > "$OUT/bench_ref.json" 2> "$OUT/bench_ref.err"; echo "bench-ref rc=$?" >> "$OUT/status.txt"
TABLE=$(python -c "import json,sys; t=json.load(open('$OUT/bench.json'))['config'].get('inc_schedule_table') or {}; print(','.join(f'{k}={v}' for k,v in t.items()))" 2>/dev/null)
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file "$OUT/launches.csv" \
    python bench.py --steps 2 --warmup 1 --no-cpu ${TABLE:+--schedule-table $TABLE} > "$OUT/bench_ncu.log" 2>&1; echo "ncu-list rc=$?" >> "$OUT/status.txt"
timeout 900 ncu --set full --clock-control none --import-source on --kernel-name-base demangled \
    -k "regex:k_gather|k_pfold|k_direct" -s 0 -c 20 \
    -o "$OUT/edge_loops" python scripts/profile_proxy.py --iters 1 --inc-schedule gather pfold > "$OUT/ncu_full.log" 2>&1; echo "ncu-full rc=$?" >> "$OUT/status.txt"
cat "$OUT/status.txt"
tail -3 "$OUT/pytest_gpu.log"
cat "$OUT/schedules.log"
cat "$OUT/bench.json"
