#!/bin/bash
# r02a: first GPU pass of round 2 -- tests, smoke, default bench (configs[4]
# BFS scale 28), its launch list, the host's memory/cores, a full ncu capture
# of k_bfs_coop at scale 28.
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
tag=r02a
(free -g; nproc; nvidia-smi --query-gpu=name,memory.total,clocks.max.sm --format=csv) > gpurun_out/${tag}_host.txt 2>&1
timeout 2400 python -m pytest tests -m gpu -x -q > gpurun_out/${tag}_gpu_tests.log 2>&1; echo "tests rc=$?" >> gpurun_out/${tag}_gpu_tests.log
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/${tag}_smoke.log 2>&1
timeout 1200 python bench.py > gpurun_out/${tag}_bench_bfs28.json 2> gpurun_out/${tag}_bench_bfs28.err
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 3000 --csv \
  --log-file gpurun_out/${tag}_bench_bfs28_launches.csv python bench.py --steps 2 --warmup 1 --no-cpu-baseline \
  > gpurun_out/${tag}_ncu_launch_bfs28.log 2>&1
timeout 1200 ncu --set full --import-source on --clock-control none -k regex:k_bfs_coop -s 1 -c 1 \
  -o gpurun_out/${tag}_bfs28_coop python tools/prof_run.py bfs --scale 28 --reps 2 > gpurun_out/${tag}_ncu_bfs28.log 2>&1
tail -3 gpurun_out/${tag}_gpu_tests.log; cat gpurun_out/${tag}_smoke.log; cat gpurun_out/${tag}_host.txt
python -c "import json,sys; d=json.loads(open(sys.argv[1]).read().strip().splitlines()[-1]); print(d.get('value'), d.get('ms_per_step'), d.get('roofline'), d.get('e2e'), d.get('cpu_baseline'))" gpurun_out/${tag}_bench_bfs28.json || tail -5 gpurun_out/${tag}_bench_bfs28.err
ls -la gpurun_out/${tag}_*
