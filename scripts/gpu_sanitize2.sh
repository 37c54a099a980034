#!/bin/bash
OUT=gpurun_out; mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build()" > $OUT/build_san2.log 2>&1 || { echo BUILD FAILED; exit 1; }
for tool in memcheck racecheck synccheck; do
timeout 1500 compute-sanitizer --tool $tool python scripts/sanitize_case2.py > $OUT/san2_$tool.log 2>&1; echo "$tool rc=$?"; tail -2 $OUT/san2_$tool.log
done
