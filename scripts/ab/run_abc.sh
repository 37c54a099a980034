#!/bin/bash
set -u
OUT=gpurun_out; mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build()" > /tmp/b.log 2>&1 || { tail /tmp/b.log; exit 1; }
cp paper_2111_10270_b200/libfastdog.so /tmp/libA.so
bash scripts/ab/build_variant.sh scripts/ab/kernels_B.cu /tmp/libB.so
bash scripts/ab/build_variant.sh scripts/ab/kernels_C.cu /tmp/libC.so
for rep in 1 2; do
for v in A B C; do for w in ${WL:-mrf_potts mrf_potts_cut gm_worms_like}; do
FDOG_LIB=/tmp/lib$v.so timeout 600 python bench.py --steps 30 --warmup 5 --no-cpu --no-hop --no-e2e --no-ttl --no-traffic --workload $w > $OUT/abc_${v}_${w}_$rep.json 2>/dev/null
python -c "
import json; d=json.load(open('$OUT/abc_${v}_${w}_$rep.json'))
print('$rep $v $w', round(d['ms_per_step'],4), {k: round(v['ms']/v['launches']*1e3,1) for k,v in d['kernels'].items()})"
done; done; done
