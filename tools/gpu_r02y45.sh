#!/bin/bash
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
for cap in 0 64 16; do
GM_WALK_CAP=$cap timeout 900 python bench.py --sharded --no-cpu-baseline --steps 3 > gpurun_out/y45_$cap.json 2>/dev/null
python -c "
import json; d=json.loads(open('gpurun_out/y45_$cap.json').read().strip().splitlines()[-1]); print('cap $cap', d['value'], d['ms_per_step'], [(x['it'], x['us']) for x in d.get('per_superstep',[]) if x['us']>50])"
done
