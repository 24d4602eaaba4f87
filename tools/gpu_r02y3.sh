#!/bin/bash
# BFS output-pass change: BFS GPU tests + bfs28 / bfs23 bench lines
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q -k "bfs or traversal or isolated" > gpurun_out/y5_tests.log 2>&1; echo "rc=$?" >> gpurun_out/y5_tests.log
tail -5 gpurun_out/y5_tests.log
timeout 600 python bench.py --no-cpu-baseline > gpurun_out/y5_bfs28.json 2> gpurun_out/y5_bfs28.err
timeout 600 python bench.py --workload bfs --no-cpu-baseline > gpurun_out/y5_bfs23.json 2> gpurun_out/y5_bfs23.err
cut -c1-400 gpurun_out/y5_bfs28.json gpurun_out/y5_bfs23.json
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_requests_srcunit_tex.sum --clock-control none -k regex:k_bfs_output -c 3 --csv python bench.py --steps 2 --warmup 1 --no-cpu-baseline > gpurun_out/y5_out_ncu.csv 2>&1
grep k_bfs_output gpurun_out/y5_out_ncu.csv | head -12
