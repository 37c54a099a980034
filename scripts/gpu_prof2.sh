#!/bin/bash
# ncu full captures of the forward sweep for several (workload, design) pairs.
OUT=gpurun_out; mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build()" > $OUT/build_p2.log 2>&1 || { echo BUILD FAILED; exit 1; }
for wm in ${CASES:-gm_worms_like:tma celltrack:rc}; do
w=${wm%%:*}; m=${wm##*:}
FDOG_SWEEP=$m timeout 900 ncu --set full --clock-control none --import-source on -k regex:"sweep" -s 4 -c 2 -o $OUT/prof_${w}_$m python bench.py --steps 2 --warmup 3 --no-cpu --no-e2e --no-ttl --workload $w > $OUT/ncu_${w}_$m.log 2>&1; echo "ncu $w $m rc=$?"; tail -2 $OUT/ncu_${w}_$m.log
done
