#!/usr/bin/env bash
# GPU tests + a profile_proxy sweep + ncu of kernels matching NCU_RE.
#   SWEEP="--inc-schedule gather pfold" NCU_RE=k_gather NCU_ARGS="--inc-schedule gather" gpurun -- bash scripts/gpu_sweep2.sh <tag>
set -u
TAG=${1:-sweep}
OUT=gpurun_out/$TAG; mkdir -p "$OUT"
python -c "import __graft_entry__ as g; g.build()" > "$OUT/build.log" 2>&1
if [ -z "${NOTEST:-}" ]; then
timeout 900 python -m pytest tests -q -m gpu -p no:cacheprovider -x > "$OUT/pytest_gpu.log" 2>&1; echo "pytest rc=$?" >> "$OUT/status.txt"
fi
timeout 900 python scripts/profile_proxy.py --iters 3 ${SWEEP:-} > "$OUT/schedules.log" 2>&1; echo "sched rc=$?" >> "$OUT/status.txt"
if [ -n "${NCU_RE:-}" ]; then
timeout 600 ncu --set full --clock-control none --import-source on --kernel-name-base demangled \
   -k "regex:${NCU_RE}" -s 0 -c ${NCU_COUNT:-3} -o "$OUT/prof" \
   python scripts/profile_proxy.py --iters 1 ${NCU_ARGS:-} > "$OUT/ncu.log" 2>&1; echo "ncu rc=$?" >> "$OUT/status.txt"
fi
cat "$OUT/status.txt"; tail -3 "$OUT/pytest_gpu.log" 2>/dev/null; cat "$OUT/schedules.log"
