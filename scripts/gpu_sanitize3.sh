#!/bin/bash
OUT=gpurun_out; mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build()" > $OUT/build_san3.log 2>&1 || { echo BUILD FAILED; exit 1; }
for tool in memcheck racecheck synccheck; do
timeout 1500 compute-sanitizer --tool $tool python scripts/sanitize_case3.py > $OUT/san3_$tool.log 2>&1; echo "$tool rc=$?"; tail -2 $OUT/san3_$tool.log
done
