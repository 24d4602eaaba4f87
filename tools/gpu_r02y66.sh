#!/bin/bash
# PageRank scale 20 / 23: hub window sweep
cd "$(dirname "$0")/.."
for w in pagerank pagerank23; do
for cap in 49152 32768 16384 8192; do
  GM_PR_HUBCAP=$cap timeout 600 python bench.py --workload $w --no-cpu-baseline --steps 10 > gpurun_out/y66_${w}_$cap.json 2>/dev/null
  python -c "import json; d=json.loads(open('gpurun_out/y66_${w}_$cap.json').read().strip().splitlines()[-1]); print('$w cap $cap', d['value'], d['ms_per_step'], d['roofline']['launch_us'])"
done
done
