#!/bin/bash
# non-deferred variant: GPU tests + deferred vs sequential comparison per workload
OUT=gpurun_out; mkdir -p $OUT
TAG=${TAG:-sq}
python -c "import __graft_entry__ as g; g.build()" > $OUT/build_$TAG.log 2>&1 || { echo BUILD FAILED; exit 1; }
timeout 900 python -m pytest tests/test_gpu_seq.py -x -q > $OUT/pytest_$TAG.log 2>&1; echo "pytest seq rc=$?"; tail -3 $OUT/pytest_$TAG.log
for w in ${WORKLOADS:-gm_worms_like celltrack qap50}; do
timeout 900 python bench.py --steps 10 --warmup 3 --no-cpu --no-e2e --seq-compare --workload $w > $OUT/bench_${TAG}_$w.json 2> $OUT/bench_${TAG}_$w.err; echo "bench $w rc=$?"
python -c "
import json; d=json.load(open('$OUT/bench_${TAG}_$w.json')); s=d['seq_compare']; t=d['time_to_lb']
print('$w deferred: %.1f us/it, ttl %.4f s / %d it | seq: %.1f us/it, ttl %.4f s / %d it reached %s' % (d['ms_per_step']*1e3, t['seconds'], t['iterations'], s['ms_per_iteration']*1e3, s['time_to_lb']['seconds'], s['time_to_lb']['iterations'], s['time_to_lb']['reached']))" || tail -5 $OUT/bench_${TAG}_$w.err
done
