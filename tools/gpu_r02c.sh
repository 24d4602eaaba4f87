#!/bin/bash
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
tag=r02c
timeout 600 python -m pytest -m gpu -q -x tests/test_gpu_dist.py > gpurun_out/${tag}_tests.log 2>&1; echo "rc=$?" >> gpurun_out/${tag}_tests.log
for w in bfs28 pagerank28; do
  timeout 900 python bench.py --workload $w --sharded --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/${tag}_bench_${w}_sharded.json 2> gpurun_out/${tag}_bench_${w}_sharded.err
done
timeout 900 python bench.py --workload pagerank28 --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/${tag}_bench_pagerank28.json 2> gpurun_out/${tag}_bench_pagerank28.err
tail -3 gpurun_out/${tag}_tests.log
for f in gpurun_out/${tag}_bench_*.json; do echo $f; python -c "import json,sys; d=json.loads(open(sys.argv[1]).read().strip().splitlines()[-1]); print(d.get('value'), d.get('ms_per_step'), d.get('config',{}).get('parallelism'), (d.get('roofline') or {}).get('frac'), d.get('e2e'), d.get('graph'))" $f || tail -5 ${f%.json}.err; done
