#!/bin/bash
# output-pass batch sweep at scale 28 (bench ms_per_step)
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
for B in 4 8 16 32; do
  GM_BFS_OUT_BATCH=$B timeout 300 python bench.py --no-cpu-baseline --steps 20 > gpurun_out/y6_b$B.json 2>/dev/null
  python -c "import json; d=json.loads(open('gpurun_out/y6_b$B.json').read().strip().splitlines()[-1]); print('B=$B', d['value'], d['ms_per_step'])"
done
