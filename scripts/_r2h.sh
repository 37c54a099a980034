set -u
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build_r2n.log 2>&1 || { tail gpurun_out/build_r2n.log; exit 1; }
timeout 1500 python -m pytest tests -q -m gpu -x > gpurun_out/pytest_r2n.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/pytest_r2n.log
WL="qap50 mrf_potts celltrack gm_worms_like mrf_potts_cut" bash scripts/gpu_ab_tree.sh r2n
