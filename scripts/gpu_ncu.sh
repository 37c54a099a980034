#!/bin/bash
# ncu --set full of one forward sweep and one averaging launch per workload.
# Usage: scripts/gpu_ncu.sh TAG "workloads"   (reports: gpurun_out/prof_TAG_<w>_<kernel>.ncu-rep)
set -u
TAG=$1; WL=${2:-celltrack qap50}
OUT=gpurun_out; mkdir -p $OUT
[ -f paper_2111_10270_b200/libfastdog.so ] || python -c "import __graft_entry__ as g; g.build()" > $OUT/build_$TAG.log 2>&1 || { tail -20 $OUT/build_$TAG.log; exit 1; }
for w in $WL; do
  for ks in ${KERNELS:-sweep_kernel:5 avg_kernel:4}; do
    k=${ks%%:*}; sk=${ks##*:}
    timeout 900 ncu --set full --clock-control none --import-source on -k regex:"$k" -s $sk -c 1 -o $OUT/prof_${TAG}_${w}_${k%%_*} python bench.py --steps 2 --warmup 3 --no-cpu --no-e2e --no-ttl --no-traffic --no-hop --workload $w > $OUT/ncu_${TAG}_${w}_${k%%_*}.log 2>&1; echo "ncu $w $k rc=$?"
    # (reports stay on the box: gpurun_out/ comes back only under 64 MiB) raw metrics + source hotspots
    R=$OUT/prof_${TAG}_${w}_${k%%_*}
    ncu -i $R.ncu-rep --page raw --csv > $R.raw.csv 2>/dev/null
    ncu -i $R.ncu-rep --page source --csv --print-source sass 2>/dev/null | gzip > $R.sass.csv.gz
    mv $R.ncu-rep /tmp/ 2>/dev/null
  done
done
