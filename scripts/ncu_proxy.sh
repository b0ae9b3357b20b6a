#!/usr/bin/env bash
# ncu captures of the proxy edge loops. Usage: gpurun -- bash scripts/ncu_proxy.sh TAG [regex] [extra args]
set -u
TAG=${1:-prof}; RE=${2:-ProxyVflux|ProxyGrad|ProxyIflux}; shift; [ $# -gt 0 ] && shift
OUT=gpurun_out/$TAG; mkdir -p "$OUT"
python -c "import __graft_entry__ as g; g.build()" > "$OUT/build.log" 2>&1
timeout 300 python scripts/profile_proxy.py --iters 2 "$@" > "$OUT/eager.log" 2>&1
timeout 900 ncu --set full --clock-control none --import-source on --kernel-name-base demangled \
   -k "regex:$RE" -s 3 -c 6 -o "$OUT/full" python scripts/profile_proxy.py --iters 1 "$@" > "$OUT/ncu_full.log" 2>&1
echo "ncu rc=$?" >> "$OUT/status.txt"
cat "$OUT/eager.log"; tail -3 "$OUT/ncu_full.log"
