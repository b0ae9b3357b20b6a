set -u
OUT=gpurun_out/${1:-kd}; mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build()" > $OUT/build.log 2>&1
timeout 900 python scripts/profile_proxy.py --iters 3 --inc-schedule gather --own-kb 0 96 48 > $OUT/cm.log 2>&1
timeout 900 python scripts/profile_proxy.py --iters 3 --kd 8 --inc-schedule gather --own-kb 0 96 48 >> $OUT/kd.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on --kernel-name-base demangled -k "regex:k_gather" -s 0 -c 3 -o $OUT/prof python scripts/profile_proxy.py --iters 1 --kd 8 --inc-schedule gather --own-kb 96 > $OUT/ncu.log 2>&1
cat $OUT/cm.log $OUT/kd.log
