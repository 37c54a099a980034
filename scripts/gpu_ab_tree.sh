#!/bin/bash
# Same-box A/B of two whole trees: this one (new) and the tree under $OLD
# (e.g. a `git worktree` of an earlier commit, built, copied to build/ab/old);
# both libraries are the ones built in this container (no rebuild on the box).
# Usage: OLD=build/ab/old WL="gm_worms_like celltrack" scripts/gpu_ab_tree.sh TAG
set -u
TAG=$1; OLD=${OLD:-build/ab/old}
OUT=$PWD/gpurun_out; mkdir -p $OUT
# (both trees built HERE beforehand: builds on different hosts differ in SASS)
cuobjdump -sass paper_2111_10270_b200/libfastdog.so | md5sum > $OUT/abt_md5_$TAG.txt
for rep in 1 2; do
for w in ${WL:-gm_worms_like celltrack qap50}; do
for arm in old new; do
  if [ $arm = old ]; then D=$OLD; else D=.; fi
  (cd $D && timeout 600 python bench.py --steps 30 --warmup 5 --no-cpu --no-hop --no-e2e --no-ttl --no-traffic --workload $w > $OUT/abt_${TAG}_${arm}_${w}_$rep.json 2>/dev/null)
  python -c "
import json; d=json.load(open('$OUT/abt_${TAG}_${arm}_${w}_$rep.json'))
print('$rep $arm $w', round(d['ms_per_step']*1e3,1), {k: round(v['ms']/v['launches']*1e3,1) for k,v in d['kernels'].items()})" || echo "$rep $arm $w failed"
done; done; done
