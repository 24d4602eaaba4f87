#!/bin/bash
cd "$(dirname "$0")/.."
for v in "" 1; do
GM_DB_PERSIST=$v timeout 900 python bench.py --sharded --no-cpu-baseline --steps 3 > gpurun_out/y50_$v.json 2>gpurun_out/y50_$v.err
python -c "
import json; d=json.loads(open('gpurun_out/y50_$v.json').read().strip().splitlines()[-1]); print('persist=$v', d['value'], d['ms_per_step'], [(x['it'], x['us']) for x in d.get('per_superstep',[]) if x['us']>50])" || tail -3 gpurun_out/y50_$v.err
done
