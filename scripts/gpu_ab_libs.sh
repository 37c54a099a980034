#!/bin/bash
# Same-box A/B/... of library variants built in this container (FDOG_LIB).
# Usage: LIBS="build/ab/var/libA.so build/ab/var/libB.so" WL="..." scripts/gpu_ab_libs.sh TAG
set -u
TAG=$1
OUT=gpurun_out; mkdir -p $OUT
for rep in 1 2; do
for w in ${WL:-mrf_potts}; do
for lib in $LIBS; do
  v=$(basename $lib .so)
  FDOG_LIB=$PWD/$lib timeout 600 python bench.py --steps 30 --warmup 5 --no-cpu --no-hop --no-e2e --no-ttl --no-traffic --workload $w > $OUT/abl_${TAG}_${v}_${w}_$rep.json 2>/dev/null
  python -c "
import json; d=json.load(open('$OUT/abl_${TAG}_${v}_${w}_$rep.json'))
print('$rep $v $w', round(d['ms_per_step']*1e3,1), {k: round(v['ms']/v['launches']*1e3,1) for k,v in d['kernels'].items()})" || echo "$rep $v $w failed"
done; done; done
