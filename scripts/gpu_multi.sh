#!/usr/bin/env bash
# Multi-rank checks on one GPU: device multi-rank tests + a 2-process bench (gloo transport).
set -u
TAG=${1:-multi}; shift || true
OUT=gpurun_out/$TAG; mkdir -p "$OUT"
python -c "import __graft_entry__ as g; g.build()" > "$OUT/build.log" 2>&1
timeout 900 python -m pytest tests/test_multigpu_device.py -q -m gpu -p no:cacheprovider -x > "$OUT/pytest_multi.log" 2>&1; echo "pytest-multi rc=$?" >> "$OUT/status.txt"
ML_TRANSPORT=gloo ML_DEVICE=0 CUDA_VISIBLE_DEVICES=0 timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 \
   --master-addr 127.0.0.1 --master-port 29533 bench.py --gpus 2 --steps 5 --warmup 2 --grid 60 > "$OUT/bench2.json" 2> "$OUT/bench2.err"; echo "bench2 rc=$?" >> "$OUT/status.txt"
cat "$OUT/status.txt"; tail -3 "$OUT/pytest_multi.log"; cat "$OUT/bench2.json"; tail -5 "$OUT/bench2.err"
