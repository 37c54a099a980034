#!/bin/bash
OUT=gpurun_out; mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build()" > $OUT/build_san.log 2>&1 || { echo BUILD FAILED; exit 1; }
for tool in memcheck racecheck synccheck; do
timeout 1200 compute-sanitizer --tool $tool python scripts/sanitize_case.py > $OUT/san_$tool.log 2>&1; echo "$tool rc=$?"; tail -2 $OUT/san_$tool.log
done
