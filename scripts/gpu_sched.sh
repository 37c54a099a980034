#!/bin/bash
OUT=gpurun_out; mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1 || exit 1
for sc in ${SCHEDS:-dynamic static}; do for w in ${WORKLOADS:-gm_worms_like}; do
FDOG_SCHED=$sc timeout 600 python bench.py --steps 30 --warmup 5 --no-cpu --no-e2e --no-ttl --workload $w > $OUT/bench_s_${w}_$sc.json 2>&1
python -c "
import json; d=json.load(open('$OUT/bench_s_${w}_$sc.json'))
print('$sc $w value %.3e ms/step %.4f roof %.3f' % (d['value'], d['ms_per_step'], d['roofline']['frac']), {k: round(v['ms']/v['launches']*1e3,2) for k,v in d['kernels'].items()})" || tail -3 $OUT/bench_s_${w}_$sc.json
done; done
