#!/bin/bash
# bench the GM workload with 1 and 2 stage buffers per warp
TAG=${1:-nb}
OUT=gpurun_out; mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build()" > $OUT/build_$TAG.log 2>&1 || { echo BUILD FAILED; tail $OUT/build_$TAG.log; exit 1; }
timeout 900 python -m pytest tests -x -q -m gpu > $OUT/pytest_gpu_$TAG.log 2>&1; echo "pytest gpu rc=$?"; tail -5 $OUT/pytest_gpu_$TAG.log
for nb in 2 1; do for w in ${WORKLOADS:-gm_worms_like}; do
FDOG_NBUF=$nb timeout 600 python bench.py --steps 30 --warmup 5 --no-cpu --no-e2e --no-ttl --workload $w > $OUT/bench_${TAG}_${w}_$nb.json 2>&1
python -c "
import json; d=json.load(open('$OUT/bench_${TAG}_${w}_$nb.json'))
print('nb=$nb $w value %.3e ms/step %.4f roof %.3f' % (d['value'], d['ms_per_step'], d['roofline']['frac']), {k: round(v['ms']/v['launches']*1e3,2) for k,v in d['kernels'].items()}, d['solver_stats']['sweep_smem_per_warp'], d['solver_stats']['sweep_grid'])" || tail -5 $OUT/bench_${TAG}_${w}_$nb.json
done; done
