#!/bin/bash
# Same-box A/B of an environment knob: bench lines of WL with and without it.
# Usage: scripts/gpu_ab.sh TAG "ENV=VAL" "workloads"
set -u
TAG=$1; ENVB=$2; WL=$3
OUT=gpurun_out; mkdir -p $OUT
for w in $WL; do
  for arm in A B; do
    if [ $arm = A ]; then E=""; else E="$ENVB"; fi
    env $E timeout 900 python bench.py --steps 30 --warmup 5 --no-cpu --no-hop --no-e2e --no-ttl --no-traffic --workload $w > $OUT/ab_${TAG}_${w}_$arm.json 2> $OUT/ab_${TAG}_${w}_$arm.err
    python -c "
import json; d=json.load(open('$OUT/ab_${TAG}_${w}_$arm.json'))
print('$arm $w [$E] ms/step %.4f value %.3e roof %.3f' % (d['ms_per_step'], d['value'], d['roofline']['frac']), {k: round(v['ms']/v['launches']*1e3,2) for k,v in d['kernels'].items()})" || tail -3 $OUT/ab_${TAG}_${w}_$arm.err
  done
done
