#!/bin/bash
# bench every (sweep design, stage buffers) pair per workload; then the GPU suite
TAG=${1:-m2}
OUT=gpurun_out; mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build()" > $OUT/build_$TAG.log 2>&1 || { echo BUILD FAILED; tail $OUT/build_$TAG.log; exit 1; }
for w in ${WORKLOADS:-gm_worms_like mrf_potts celltrack qap50}; do for mode in ${MODES:-rc:1 rc:2 tma:1 tma:2 stream:2}; do
m=${mode%%:*}; nb=${mode##*:}
FDOG_SWEEP=$m FDOG_NBUF=$nb timeout 600 python bench.py --steps 30 --warmup 5 --no-cpu --no-e2e --no-ttl --workload $w > $OUT/bench_${TAG}_${w}_${m}$nb.json 2>&1
python -c "
import json; d=json.load(open('$OUT/bench_${TAG}_${w}_${m}$nb.json'))
print('$m nb$nb $w value %.3e ms/step %.4f roof %.3f' % (d['value'], d['ms_per_step'], d['roofline']['frac']), {k: round(v['ms']/v['launches']*1e3,2) for k,v in d['kernels'].items()}, d['solver_stats'].get('sweep_smem_per_warp'), d['solver_stats'].get('sweep_grid'))" || tail -5 $OUT/bench_${TAG}_${w}_${m}$nb.json
done; done
if [ -z "${NOTEST:-}" ]; then timeout 1500 python -m pytest tests -x -q -m gpu > $OUT/pytest_gpu_$TAG.log 2>&1; echo "pytest gpu rc=$?"; tail -5 $OUT/pytest_gpu_$TAG.log; fi
