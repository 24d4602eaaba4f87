#!/bin/bash
# Re-entry check: GPU tests, smoke, default bench line and the per-workload lines.
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
tag=${1:-r02q}
timeout 2400 python -m pytest tests -m gpu -q > gpurun_out/${tag}_gpu_tests.log 2>&1; echo "tests rc=$?" >> gpurun_out/${tag}_gpu_tests.log
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/${tag}_smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/${tag}_smoke.log
timeout 1200 python bench.py > gpurun_out/${tag}_bench_bfs28.json 2> gpurun_out/${tag}_bench_bfs28.err
for w in ${WORKLOADS:-bfs pagerank23 pagerank28 cf}; do
  timeout 900 python bench.py --workload $w --no-cpu-baseline > gpurun_out/${tag}_bench_$w.json 2> gpurun_out/${tag}_bench_$w.err
done
tail -3 gpurun_out/${tag}_gpu_tests.log; cat gpurun_out/${tag}_smoke.log
for f in gpurun_out/${tag}_bench_*.json; do echo "== $f"; tail -1 $f | cut -c1-600; done
