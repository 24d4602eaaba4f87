#!/bin/bash
# BFS iteration: parity tests, bench bfs28 + bfs (23), per-superstep phases
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
tag=$1
timeout 900 python -m pytest -m gpu -q -x tests/test_gpu_configs.py::test_config1_bfs_scale23 tests/test_gpu_scale28.py::test_config4_bfs_scale28_invariants tests/test_gpu_parity.py -k "bfs or golden or BFS" > gpurun_out/${tag}_tests.log 2>&1; echo "rc=$?" >> gpurun_out/${tag}_tests.log
timeout 900 python bench.py --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/${tag}_bench_bfs28.json 2> gpurun_out/${tag}_bench_bfs28.err
timeout 900 python bench.py --workload bfs --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/${tag}_bench_bfs23.json 2> gpurun_out/${tag}_bench_bfs23.err
GM_BFS_PHASES=1 timeout 600 python -c "
import paper_1503_07241_b200 as gm
g = gm.Graph.rmat(28, 16, seed=1, symmetrize=True, relabel=True, a=0.57, b=0.19, c=0.19)
r = g.pick_source(1)
for _ in range(2): gm.bfs(g, r)
" > gpurun_out/${tag}_phases28.log 2>&1
GM_BFS_PHASES=1 timeout 600 python -c "
import paper_1503_07241_b200 as gm
g = gm.Graph.rmat(23, 16, seed=1, symmetrize=True, relabel=True, a=0.57, b=0.19, c=0.19)
r = g.pick_source(1)
for _ in range(3): gm.bfs(g, r)
" > gpurun_out/${tag}_phases23.log 2>&1
tail -3 gpurun_out/${tag}_tests.log
for f in gpurun_out/${tag}_bench_*.json; do echo $f; python -c "
import json,sys; d=json.loads(open(sys.argv[1]).read().strip().splitlines()[-1]); print(d.get('value'), d.get('ms_per_step'), (d.get('roofline') or {}).get('frac'), (d.get('roofline') or {}).get('launch_us'), d.get('e2e',{}).get('value'))
for s in d['per_superstep']: print('  ', s)" $f || tail -5 ${f%.json}.err; done
tail -12 gpurun_out/${tag}_phases28.log
tail -16 gpurun_out/${tag}_phases23.log
