#!/bin/bash
# bench one workload list under several environment settings: ENVSETS="A=1,B=2 A=2" (comma = several vars)
OUT=gpurun_out; mkdir -p $OUT
TAG=${TAG:-e}
python -c "import __graft_entry__ as g; g.build()" > $OUT/build_$TAG.log 2>&1 || { echo BUILD FAILED; tail $OUT/build_$TAG.log; exit 1; }
for w in ${WORKLOADS:-gm_worms_like celltrack qap50}; do for es in ${ENVSETS:-X=0}; do
f=$OUT/bench_${TAG}_${w}_$(echo $es | tr ',=' '__').json
env $(echo $es | tr ',' ' ') timeout 600 python bench.py --steps 30 --warmup 5 --no-cpu --no-e2e --no-ttl --workload $w > $f 2>&1
python -c "
import json; d=json.load(open('$f'))
print('$es $w ms/step %.4f' % (d['ms_per_step']), {k: round(v['ms']/v['launches']*1e3,2) for k,v in d['kernels'].items()}, d['solver_stats'].get('sweep_grid'), d['solver_stats'].get('sweep_block'))" || tail -5 $f
done; done
