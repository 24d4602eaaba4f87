#!/bin/bash
# A/B of GM_DB_HEAD0 (dense first-neighbour array in the sharded BFS pull):
# the sharded GPU tests with it on, then the sharded bench at scales 28 and 23.
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
GM_DB_HEAD0=1 timeout 1500 python -m pytest tests/test_gpu_dist.py tests/test_gpu_checked.py -m gpu -q > gpurun_out/r02t_dist_tests_head0.log 2>&1; echo "tests rc=$?" >> gpurun_out/r02t_dist_tests_head0.log
for h in 0 1 0 1; do
  GM_DB_HEAD0=$h timeout 900 python bench.py --sharded --no-cpu-baseline >> gpurun_out/r02t_sharded_bfs28_head$h.json 2>> gpurun_out/r02t_sharded.err
done
for h in 0 1; do
  GM_DB_HEAD0=$h timeout 900 python bench.py --sharded --workload bfs --no-cpu-baseline >> gpurun_out/r02t_sharded_bfs23_head$h.json 2>> gpurun_out/r02t_sharded.err
done
GM_DB_HEAD0=0 timeout 600 python -m pytest tests/test_gpu_dist.py -m gpu -q > gpurun_out/r02t_gpu_tests.log 2>&1; echo "tests rc=$?" >> gpurun_out/r02t_gpu_tests.log
python -c "import __graft_entry__ as g; g.smoke()" >> gpurun_out/r02t_gpu_tests.log 2>&1
tail -n 4 gpurun_out/r02t_dist_tests_head0.log gpurun_out/r02t_gpu_tests.log
python - <<'P'
import json,glob
for f in sorted(glob.glob('gpurun_out/r02t_sharded_bfs*_head*.json')):
    for line in open(f):
        try: d=json.loads(line)
        except Exception: continue
        print(f[11:], d['value'], d['ms_per_step'], [(p['dir'][:2], p['us']) for p in d.get('per_superstep',[])])
P
tail -n 5 gpurun_out/r02t_sharded.err
