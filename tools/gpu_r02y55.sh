#!/bin/bash
cd "$(dirname "$0")/.."
for v in ${VALS:-1 4 8 16 64}; do
  GM_BFS_HV_DIV=$v timeout 600 python bench.py --no-cpu-baseline --steps 10 > gpurun_out/y55_$v.json 2>/dev/null
  python -c "import json; d=json.loads(open('gpurun_out/y55_$v.json').read().strip().splitlines()[-1]); print('hv_div $v', d['value'], d['ms_per_step'], [(x['it'], x['us']) for x in d['per_superstep'] if x['us']>50])"
  GM_BFS_HV_DIV=$v timeout 600 python bench.py --workload bfs --no-cpu-baseline --steps 10 > gpurun_out/y55_23_$v.json 2>/dev/null
  python -c "import json; d=json.loads(open('gpurun_out/y55_23_$v.json').read().strip().splitlines()[-1]); print('  23: hv_div $v', d['value'], d['ms_per_step'])"
done
