#!/bin/bash
# sharded BFS change: dist + sharded GPU tests, checked build tests, --sharded bench at scale 28
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
T=${1:-y26}
timeout 1200 python -m pytest tests -m gpu -x -q -k "dist or dgraph or sharded or checked" > gpurun_out/${T}_tests.log 2>&1; echo "rc=$?" >> gpurun_out/${T}_tests.log
tail -4 gpurun_out/${T}_tests.log
timeout 900 python bench.py --sharded --no-cpu-baseline --steps 5 > gpurun_out/${T}_sharded.json 2> gpurun_out/${T}_sharded.err
python -c "
import json; d=json.loads(open('gpurun_out/${T}_sharded.json').read().strip().splitlines()[-1]); print(d['value'], d['ms_per_step'], d['e2e']['value']); [print(x) for x in d.get('per_superstep',[])]"
