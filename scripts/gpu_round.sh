#!/bin/bash
# One GPU session: tests, smoke, bench, ncu launch list (+ optional full capture).
# Usage: scripts/gpu_round.sh [tag] [full]
set -u
TAG=${1:-r1}
OUT=gpurun_out
mkdir -p $OUT
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,memory.total --format=csv > $OUT/gpu_$TAG.txt 2>&1
python -c "import __graft_entry__ as g; g.build()" > $OUT/build_$TAG.log 2>&1 || { echo BUILD FAILED; tail -30 $OUT/build_$TAG.log; }
timeout 900 python -m pytest tests -x -q -m gpu > $OUT/pytest_gpu_$TAG.log 2>&1; echo "pytest gpu rc=$?"; tail -15 $OUT/pytest_gpu_$TAG.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $OUT/smoke_$TAG.log 2>&1; echo "smoke rc=$?"; tail -3 $OUT/smoke_$TAG.log
timeout 600 python bench.py --steps 50 --warmup 5 > $OUT/bench_$TAG.json 2> $OUT/bench_$TAG.err; echo "bench rc=$?"; cat $OUT/bench_$TAG.json; tail -5 $OUT/bench_$TAG.err
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file $OUT/launches_$TAG.csv python bench.py --steps 3 --warmup 3 --no-cpu --no-e2e --no-ttl > $OUT/ncu_launch_$TAG.log 2>&1; echo "ncu launches rc=$?"
if [ "${2:-}" = "full" ]; then
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:"sweep_kernel|avg_kernel" -s 8 -c 4 -o $OUT/prof_$TAG python bench.py --steps 3 --warmup 3 --no-cpu --no-e2e --no-ttl > $OUT/ncu_full_$TAG.log 2>&1; echo "ncu full rc=$?"
fi
