#!/usr/bin/env bash
# Layout x block size x schedule sweep of the proxy iteration (eager, per-loop times).
set -u
TAG=${1:-sweep}; shift || true
OUT=gpurun_out/$TAG; mkdir -p "$OUT"
python -c "import __graft_entry__ as g; g.build()" > "$OUT/build.log" 2>&1
for soa in 4 -1 0; do
  timeout 600 python scripts/profile_proxy.py --iters 3 --soa $soa --block-size 256 128 64 \
      --inc-schedule colour flow arrival "$@" >> "$OUT/sweep.log" 2>&1
done
cat "$OUT/sweep.log"
