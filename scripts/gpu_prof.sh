#!/bin/bash
# ncu full capture of the sweep kernels (1 GPU).
TAG=${1:-p}
OUT=gpurun_out
mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build()" > $OUT/build_$TAG.log 2>&1 || { echo BUILD FAILED; exit 1; }
timeout 600 python bench.py --steps 2 --warmup 3 --no-cpu --no-e2e --no-ttl ${BENCH_ARGS:-} > $OUT/bench_$TAG.json 2>&1
python -c "import json; d=json.load(open('$OUT/bench_$TAG.json')); print(d['solver_stats']); print({k: round(v['ms']/v['launches']*1e3,2) for k,v in d['kernels'].items()})"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"sweep_kernel" -s 2 -c 2 -o $OUT/prof_$TAG python bench.py --steps 2 --warmup 3 --no-cpu --no-e2e --no-ttl ${BENCH_ARGS:-} > $OUT/ncu_$TAG.log 2>&1; echo "ncu rc=$?"; tail -3 $OUT/ncu_$TAG.log
