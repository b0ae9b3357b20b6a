#!/usr/bin/env bash
# Quick GPU iteration: tests + schedule comparison + ncu of the edge loops.
#   SCHEDS="gather fold" NCU_SCHED=fold bash scripts/gpu_quick.sh <tag>
set -u
TAG=${1:-quick}
SCHEDS=${SCHEDS:-"gather fold"}
NCU_SCHED=${NCU_SCHED:-fold}
OUT=gpurun_out/$TAG; mkdir -p "$OUT"
python -c "import __graft_entry__ as g; g.build()" > "$OUT/build.log" 2>&1
timeout 900 python -m pytest tests -q -m gpu -p no:cacheprovider -x > "$OUT/pytest_gpu.log" 2>&1; echo "pytest rc=$?" >> "$OUT/status.txt"
timeout 600 python scripts/profile_proxy.py --iters 3 --inc-schedule $SCHEDS > "$OUT/schedules.log" 2>&1; echo "sched rc=$?" >> "$OUT/status.txt"
timeout 600 ncu --set full --clock-control none --import-source on --kernel-name-base demangled \
   -k "regex:Proxy(Vflux|Grad|Iflux)|k_fold_targets" -s 0 -c 6 -o "$OUT/$NCU_SCHED" \
   python scripts/profile_proxy.py --iters 1 --inc-schedule $NCU_SCHED > "$OUT/ncu.log" 2>&1; echo "ncu rc=$?" >> "$OUT/status.txt"
cat "$OUT/status.txt"; tail -2 "$OUT/pytest_gpu.log"; cat "$OUT/schedules.log"
