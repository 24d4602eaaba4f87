#!/bin/bash
# shared-memory window sweeps: SSSP pull hub copy (scale 23), BFS frontier prefix (scale 28 / 23)
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
line() { python -c "import json,sys; d=json.loads(open(sys.argv[1]).read().strip().splitlines()[-1]); print(sys.argv[2], d['value'], d['ms_per_step'])" "$@"; }
for h in 49152 32768 16384 8192; do
  GM_SSSP_HUB=$h timeout 600 python bench.py --workload sssp --no-cpu-baseline --steps 5 > gpurun_out/y32_sssp_$h.json 2>/dev/null; line gpurun_out/y32_sssp_$h.json "sssp hub $h"
done
for w in 16384 8192 4096; do
  GM_BFS_PREFIX_WORDS=$w timeout 600 python bench.py --no-cpu-baseline --steps 10 > gpurun_out/y32_bfs28_$w.json 2>/dev/null; line gpurun_out/y32_bfs28_$w.json "bfs28 prefix $w"
done
for w in 24576 16384 8192; do
  GM_BFS_PREFIX_WORDS=$w timeout 600 python bench.py --workload bfs --no-cpu-baseline --steps 10 > gpurun_out/y32_bfs23_$w.json 2>/dev/null; line gpurun_out/y32_bfs23_$w.json "bfs23 prefix $w"
done
