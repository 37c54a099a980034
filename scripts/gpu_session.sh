#!/bin/bash
# Full GPU session: build, GPU tests, smoke, default bench (MRF-LP; CPU
# baseline, e2e, time-to-LB, in-run ncu traffic), the reference-arm line,
# per-workload bench lines, ncu launch list and --set full captures (one
# forward sweep and one averaging launch per workload, small reports).
# Usage: scripts/gpu_session.sh TAG     env: WORKLOADS, FULL_WORKLOADS, SKIP_TESTS=1, TTL=1
set -u
TAG=${1:-r2}
OUT=gpurun_out; mkdir -p $OUT
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,memory.total --format=csv > $OUT/gpu_$TAG.txt 2>&1
# (the library built in this container travels with the snapshot; build here
# only if it is missing -- builds on different hosts differ in SASS)
[ -f paper_2111_10270_b200/libfastdog.so ] || python -c "import __graft_entry__ as g; g.build()" > $OUT/build_$TAG.log 2>&1 || { echo BUILD FAILED; tail -30 $OUT/build_$TAG.log; exit 1; }
cuobjdump -sass paper_2111_10270_b200/libfastdog.so | md5sum > $OUT/sass_md5_$TAG.txt
if [ "${TTL:-0}" = "1" ]; then timeout 900 python scripts/make_ttl_targets.py > $OUT/ttl_$TAG.log 2>&1; echo "ttl rc=$?"; cp bench_targets.json $OUT/bench_targets.json; fi
if [ "${SKIP_TESTS:-0}" != "1" ]; then
timeout 2400 python -m pytest tests -q -m gpu > $OUT/pytest_gpu_$TAG.log 2>&1; echo "pytest gpu rc=$?"; grep -E "FAILED|passed|failed" $OUT/pytest_gpu_$TAG.log | tail -5
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $OUT/smoke_$TAG.log 2>&1; echo "smoke rc=$?"; tail -1 $OUT/smoke_$TAG.log
fi
timeout 1200 python bench.py --steps 50 --warmup 5 > $OUT/bench_$TAG.json 2> $OUT/bench_$TAG.err; echo "bench rc=$?"; cut -c1-600 $OUT/bench_$TAG.json; tail -3 $OUT/bench_$TAG.err
timeout 900 python bench.py --impl reference --steps 3 --warmup 3 > $OUT/bench_${TAG}_reference.json 2> $OUT/bench_${TAG}_reference.err; echo "reference rc=$?"; cut -c1-300 $OUT/bench_${TAG}_reference.json
for w in ${WORKLOADS:-mrf_potts_cut gm_worms_like celltrack qap50 qap128 gap mckp lap4 thin_hop}; do
timeout 900 python bench.py --steps 30 --warmup 5 --no-cpu --no-hop --workload $w > $OUT/bench_${TAG}_$w.json 2> $OUT/bench_${TAG}_$w.err; echo "bench $w rc=$?"; python -c "
import json; d=json.load(open('$OUT/bench_${TAG}_$w.json'))
print('$w value %.3e ms/step %.4f roof %.3f traffic %s' % (d['value'], d['ms_per_step'], d['roofline']['frac'], d['roofline']['traffic']), {k: round(v['ms']/v['launches']*1e3,2) for k,v in d['kernels'].items()})" || tail -5 $OUT/bench_${TAG}_$w.err
done
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file $OUT/launches_$TAG.csv python bench.py --steps 3 --warmup 3 --no-cpu --no-e2e --no-ttl --no-traffic --no-hop > $OUT/ncu_launch_$TAG.log 2>&1; echo "ncu launches rc=$?"
# ncu --set full of a forward sweep and an averaging launch per workload (raw
# metrics + SASS hotspots exported on the box, reports left there)
bash scripts/gpu_ncu.sh $TAG "${FULL_WORKLOADS:-mrf_potts celltrack qap50 gm_worms_like}"
