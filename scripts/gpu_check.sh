#!/bin/bash
# GPU check: build, the whole GPU suite, quick bench lines, optional ncu --set full captures.
# Usage: scripts/gpu_check.sh TAG     env: WL (bench workloads), FULL (workloads to capture), KREGEX
set -u
TAG=${1:-c}
OUT=gpurun_out; mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build()" > $OUT/build_$TAG.log 2>&1 || { echo BUILD FAILED; tail -30 $OUT/build_$TAG.log; exit 1; }
if [ "${SKIP_TESTS:-0}" != "1" ]; then
timeout 2400 python -m pytest tests -q -m gpu ${PYTEST_ARGS:-} > $OUT/pytest_gpu_$TAG.log 2>&1; echo "pytest gpu rc=$?"; grep -E "FAILED|passed|failed" $OUT/pytest_gpu_$TAG.log | tail -8
fi
for w in ${WL:-}; do
timeout 900 python bench.py --steps 30 --warmup 5 --no-cpu --no-hop --no-e2e --no-ttl --no-traffic --workload $w > $OUT/bench_${TAG}_$w.json 2> $OUT/bench_${TAG}_$w.err; echo "bench $w rc=$?"; python -c "
import json; d=json.load(open('$OUT/bench_${TAG}_$w.json'))
print('$w value %.3e ms/step %.4f roof %.3f' % (d['value'], d['ms_per_step'], d['roofline']['frac']), {k: round(v['ms']/v['launches']*1e3,2) for k,v in d['kernels'].items()}, d['solver_stats'].get('tile_pairs'))" || tail -5 $OUT/bench_${TAG}_$w.err
done
for w in ${FULL:-}; do
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"${KREGEX:-sweep_kernel|avg_kernel}" -s 12 -c 3 -o $OUT/prof_${TAG}_$w python bench.py --steps 2 --warmup 3 --no-cpu --no-e2e --no-ttl --no-traffic --no-hop --workload $w > $OUT/ncu_full_${TAG}_$w.log 2>&1; echo "ncu full $w rc=$?"
done
