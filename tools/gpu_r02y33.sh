#!/bin/bash
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
line() { python -c "import json,sys; d=json.loads(open(sys.argv[1]).read().strip().splitlines()[-1]); print(sys.argv[2], d['value'], d['ms_per_step'])" "$@"; }
for rep in 1 2; do
for w in 24576 8192 4096 2048 1024; do
  GM_BFS_PREFIX_WORDS=$w timeout 600 python bench.py --workload bfs --no-cpu-baseline --steps 20 > gpurun_out/y33_bfs23_$w.json 2>/dev/null; line gpurun_out/y33_bfs23_$w.json "bfs23 prefix $w"
done
done
