#!/bin/bash
# BFS change check: BFS GPU tests, bench bfs28 / bfs23, per-superstep phases at scale 28
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
T=${1:-y8}
timeout 900 python -m pytest tests -m gpu -x -q -k "bfs or traversal or isolated" > gpurun_out/${T}_tests.log 2>&1; echo "rc=$?" >> gpurun_out/${T}_tests.log
tail -3 gpurun_out/${T}_tests.log
timeout 600 python bench.py --no-cpu-baseline > gpurun_out/${T}_bfs28.json 2> gpurun_out/${T}_bfs28.err
timeout 600 python bench.py --workload bfs --no-cpu-baseline > gpurun_out/${T}_bfs23.json 2> gpurun_out/${T}_bfs23.err
for f in gpurun_out/${T}_bfs28.json gpurun_out/${T}_bfs23.json; do
  python -c "import json,sys; d=json.loads(open('$f').read().strip().splitlines()[-1]); print('$f', d['value'], d['ms_per_step'], d['roofline']['launch_us'], [(x['it'], x['us']) for x in d['per_superstep']])"
done
