#!/bin/bash
# PageRank scale 28 on the hub kernel with smaller hub windows (GM_PR_HUB=1, GM_PR_HUBCAP)
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
for cap in ${CAPS:-8192 12288 24576 32768}; do
  GM_PR_HUB=1 GM_PR_HUBCAP=$cap timeout 900 python bench.py --workload pagerank28 --no-cpu-baseline --steps 2 --warmup 1 > gpurun_out/y29_pr28_$cap.json 2>/dev/null
  python -c "import json; d=json.loads(open('gpurun_out/y29_pr28_$cap.json').read().strip().splitlines()[-1]); print('cap $cap', d['value'], d['ms_per_step'], d['roofline']['launch_us'], d['roofline']['kernel'])"
done
