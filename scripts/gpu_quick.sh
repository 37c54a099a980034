#!/bin/bash
# Quick GPU check: build, selected GPU tests, bench lines of selected workloads.
# Usage: scripts/gpu_quick.sh TAG "pytest args" "workloads"
set -u
TAG=${1:-q}; TESTS=${2:-}; WL=${3:-mrf_potts}
OUT=gpurun_out; mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build()" > $OUT/build_$TAG.log 2>&1 || { echo BUILD FAILED; tail -30 $OUT/build_$TAG.log; exit 1; }
if [ -n "$TESTS" ]; then timeout 1800 python -m pytest -x -q -m gpu $TESTS > $OUT/pytest_$TAG.log 2>&1; echo "pytest rc=$?"; tail -4 $OUT/pytest_$TAG.log; fi
for w in $WL; do
timeout 900 python bench.py --steps 30 --warmup 5 --no-cpu --no-hop --no-e2e --no-ttl ${BENCH_ARGS:-} --workload $w > $OUT/bench_${TAG}_$w.json 2> $OUT/bench_${TAG}_$w.err; echo "bench $w rc=$?"; python -c "
import json; d=json.load(open('$OUT/bench_${TAG}_$w.json'))
print('$w value %.3e ms/step %.4f roof %.3f traffic %s' % (d['value'], d['ms_per_step'], d['roofline']['frac'], d['roofline']['traffic']), {k: round(v['ms']/v['launches']*1e3,2) for k,v in d['kernels'].items()}, d['solver_stats'].get('tile_pairs'))" || tail -5 $OUT/bench_${TAG}_$w.err
done
