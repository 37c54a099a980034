# Final check of a commit: GPU tests, smoke, the default bench line, the ncu
# launch list.  Usage: scripts/gpu_final.sh TAG
set -u
TAG=${1:-final}
OUT=gpurun_out; mkdir -p $OUT
cuobjdump -sass paper_2111_10270_b200/libfastdog.so | md5sum > $OUT/sass_md5_$TAG.txt
timeout 1500 python -m pytest tests -q -m gpu > $OUT/pytest_gpu_$TAG.log 2>&1; echo "pytest rc=$?"; tail -2 $OUT/pytest_gpu_$TAG.log
for i in 1 2 3; do timeout 120 python -m pytest tests/test_gpu_parity.py -q -k "device_memory or torch_memory" 2>&1 | tail -1; done
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $OUT/smoke_$TAG.log 2>&1; echo "smoke rc=$?"
timeout 1200 python bench.py --steps 50 --warmup 5 > $OUT/bench_$TAG.json 2> $OUT/bench_$TAG.err; echo "bench rc=$?"; cut -c1-400 $OUT/bench_$TAG.json
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file $OUT/launches_$TAG.csv python bench.py --steps 3 --warmup 3 --no-cpu --no-e2e --no-ttl --no-traffic --no-hop > $OUT/ncu_launch_$TAG.log 2>&1; echo "ncu launches rc=$?"
