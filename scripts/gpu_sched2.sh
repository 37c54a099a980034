#!/bin/bash
# scheduling / buffering experiments on the recompute design
OUT=gpurun_out; mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build()" > $OUT/build_s2.log 2>&1 || { echo BUILD FAILED; exit 1; }
for w in ${WORKLOADS:-gm_worms_like celltrack qap50}; do for cfg in ${CFGS:-static:1 dynamic:1 static:2 dynamic:2}; do
sc=${cfg%%:*}; nb=${cfg##*:}
FDOG_SCHED=$sc FDOG_NBUF=$nb timeout 600 python bench.py --steps 30 --warmup 5 --no-cpu --no-e2e --no-ttl --workload $w > $OUT/bench_s2_${w}_${sc}$nb.json 2>&1
python -c "
import json; d=json.load(open('$OUT/bench_s2_${w}_${sc}$nb.json'))
print('$sc nb$nb $w ms/step %.4f' % (d['ms_per_step']), {k: round(v['ms']/v['launches']*1e3,2) for k,v in d['kernels'].items()}, d['solver_stats'].get('sweep_smem_per_warp'), d['solver_stats'].get('sweep_grid'))" || tail -5 $OUT/bench_s2_${w}_${sc}$nb.json
done; done
