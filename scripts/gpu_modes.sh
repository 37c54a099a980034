#!/bin/bash
# tests + bench of the two sweep implementations (FDOG_SWEEP=tma|stream)
TAG=${1:-m}
OUT=gpurun_out; mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build()" > $OUT/build_$TAG.log 2>&1 || { echo BUILD FAILED; tail $OUT/build_$TAG.log; exit 1; }
timeout 900 python -m pytest tests -x -q -m gpu > $OUT/pytest_gpu_$TAG.log 2>&1; echo "pytest gpu rc=$?"; tail -3 $OUT/pytest_gpu_$TAG.log
for mode in ${MODES:-stream tma}; do for w in ${WORKLOADS:-gm_worms_like}; do
FDOG_SWEEP=$mode timeout 600 python bench.py --steps 30 --warmup 5 --no-cpu --no-e2e --no-ttl --workload $w > $OUT/bench_${TAG}_${w}_$mode.json 2>&1
python -c "
import json; d=json.load(open('$OUT/bench_${TAG}_${w}_$mode.json'))
print('$mode $w value %.3e ms/step %.4f roof %.3f' % (d['value'], d['ms_per_step'], d['roofline']['frac']), {k: round(v['ms']/v['launches']*1e3,2) for k,v in d['kernels'].items()})" || tail -5 $OUT/bench_${TAG}_${w}_$mode.json
done; done
