#!/usr/bin/env bash
# Tile schedule check: GPU tests, schedule/budget sweep, ncu of the tile kernels.
#   gpurun -- bash scripts/gpu_tile.sh <tag>
set -u
TAG=${1:-tile}
OUT=gpurun_out/$TAG; mkdir -p "$OUT"
python -c "import __graft_entry__ as g; g.build()" > "$OUT/build.log" 2>&1
timeout 900 python -m pytest tests -q -m gpu -p no:cacheprovider -x > "$OUT/pytest_gpu.log" 2>&1; echo "pytest rc=$?" >> "$OUT/status.txt"
timeout 600 python scripts/profile_proxy.py --iters 3 --inc-schedule tile gather --tile-smem 100 50 30 --tile-threads 256 128 > "$OUT/schedules.log" 2>&1; echo "sched rc=$?" >> "$OUT/status.txt"
timeout 600 ncu --set full --clock-control none --import-source on --kernel-name-base demangled \
   -k "regex:k_tile" -s 0 -c 3 -o "$OUT/tile" \
   python scripts/profile_proxy.py --iters 1 --inc-schedule tile > "$OUT/ncu.log" 2>&1; echo "ncu rc=$?" >> "$OUT/status.txt"
cat "$OUT/status.txt"; tail -5 "$OUT/pytest_gpu.log"; cat "$OUT/schedules.log"
