#!/bin/bash
# BFS scale 23: 3-CTA variant with small frontier prefixes vs the 2-CTA default
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
line() { python -c "import json,sys; d=json.loads(open(sys.argv[1]).read().strip().splitlines()[-1]); print(sys.argv[2], d['value'], d['ms_per_step'])" "$@"; }
timeout 600 python bench.py --workload bfs --no-cpu-baseline --steps 20 > gpurun_out/y41_def.json 2>/dev/null; line gpurun_out/y41_def.json "default (2 CTA, 4K words)"
for w in 4096 8192 16384; do
  GM_BFS_CTAS_PER_SM=3 GM_BFS_PREFIX_WORDS=$w timeout 600 python bench.py --workload bfs --no-cpu-baseline --steps 20 > gpurun_out/y41_3_$w.json 2>/dev/null; line gpurun_out/y41_3_$w.json "3 CTA prefix $w"
done
for w in 2048 4096 8192; do
  GM_BFS_PREFIX_WORDS=$w timeout 600 python bench.py --no-cpu-baseline --steps 10 > gpurun_out/y41_28_$w.json 2>/dev/null; line gpurun_out/y41_28_$w.json "scale 28 3 CTA prefix $w"
done
