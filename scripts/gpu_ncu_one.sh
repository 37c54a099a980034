set -u
OUT=gpurun_out; mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build()" > /tmp/build.log 2>&1 || { tail -20 /tmp/build.log; exit 1; }
for w in mrf_potts mrf_potts_cut; do
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"sweep_kernel" -s 14 -c 1 -o $OUT/prof_r2p_${w}_fwd python bench.py --steps 2 --warmup 3 --no-cpu --no-e2e --no-ttl --no-traffic --no-hop --workload $w > /tmp/ncu_$w.log 2>&1; echo "ncu $w rc=$?"
done
ls -la $OUT
