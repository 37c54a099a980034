#!/bin/bash
# Quick GPU iteration: build, GPU tests, bench without CPU baseline.
set -u
TAG=${1:-q}
OUT=gpurun_out
mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build()" > $OUT/build_$TAG.log 2>&1 || { echo BUILD FAILED; tail -30 $OUT/build_$TAG.log; exit 1; }
timeout 900 python -m pytest tests -x -q -m gpu ${PYTEST_K:-} > $OUT/pytest_gpu_$TAG.log 2>&1; echo "pytest gpu rc=$?"; tail -25 $OUT/pytest_gpu_$TAG.log
for w in ${WORKLOADS:-gm_worms_like}; do
timeout 600 python bench.py --steps 30 --warmup 5 --no-cpu --workload $w > $OUT/bench_${TAG}_$w.json 2> $OUT/bench_${TAG}_$w.err; echo "bench $w rc=$?"; python -c "
import json,sys; d=json.load(open('$OUT/bench_${TAG}_$w.json'))
print('value %.3e ms/step %.4f iters/s %.0f roof %.3f' % (d['value'], d['ms_per_step'], d['iters_per_s'], d['roofline']['frac']))
print({k: round(v['ms']/v['launches']*1e3,2) for k,v in d['kernels'].items()}, d['gpu_launches'])
" || tail -20 $OUT/bench_${TAG}_$w.err
done
