#!/bin/bash
# Recompute vs store sweep designs: focused tests, full GPU suite, per-design bench on each workload.
TAG=${1:-rc}
OUT=gpurun_out; mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build()" > $OUT/build_$TAG.log 2>&1 || { echo BUILD FAILED; tail $OUT/build_$TAG.log; exit 1; }
timeout 600 python -m pytest tests -x -q -m gpu -k "sweep_kernels or recompute" > $OUT/pytest_rc_$TAG.log 2>&1; echo "pytest rc-focused rc=$?"; tail -15 $OUT/pytest_rc_$TAG.log
for w in ${WORKLOADS:-gm_worms_like mrf_potts celltrack qap50}; do for mode in ${MODES:-rc tma stream}; do
FDOG_SWEEP=$mode timeout 600 python bench.py --steps 30 --warmup 5 --no-cpu --no-e2e --no-ttl --workload $w > $OUT/bench_${TAG}_${w}_$mode.json 2>&1
python -c "
import json; d=json.load(open('$OUT/bench_${TAG}_${w}_$mode.json'))
print('$mode $w value %.3e ms/step %.4f roof %.3f' % (d['value'], d['ms_per_step'], d['roofline']['frac']), {k: round(v['ms']/v['launches']*1e3,2) for k,v in d['kernels'].items()}, d['solver_stats'].get('sweep_smem_per_warp'), d['solver_stats'].get('sweep_grid'))" || tail -5 $OUT/bench_${TAG}_${w}_$mode.json
done; done
timeout 1200 python -m pytest tests -x -q -m gpu > $OUT/pytest_gpu_$TAG.log 2>&1; echo "pytest gpu rc=$?"; tail -5 $OUT/pytest_gpu_$TAG.log
