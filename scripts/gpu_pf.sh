#!/bin/bash
OUT=gpurun_out; mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1 || exit 1
for pf in 2 4; do for w in ${WORKLOADS:-qap50 celltrack}; do
FDOG_PREFETCH=$pf timeout 600 python bench.py --steps 30 --warmup 5 --no-cpu --no-e2e --no-ttl --workload $w > $OUT/bench_pf_${w}_$pf.json 2>&1
python -c "
import json; d=json.load(open('$OUT/bench_pf_${w}_$pf.json'))
print('pf=$pf $w value %.3e ms/step %.4f roof %.3f' % (d['value'], d['ms_per_step'], d['roofline']['frac']), {k: round(v['ms']/v['launches']*1e3,2) for k,v in d['kernels'].items()})" || tail -3 $OUT/bench_pf_${w}_$pf.json
done; done
