mkdir -p gpurun_out
timeout 600 python -m pytest tests -m gpu -q -x -k "pagerank or shard or smoke" 2>&1 | tail -5 > gpurun_out/t.log
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:k_pr -c 20 --csv --log-file gpurun_out/z.csv python tools/pr_once.py 23 > /dev/null 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:k_pr -c 20 --csv --log-file gpurun_out/z_stats.csv python tools/pr_once.py 23 stats > /dev/null 2>&1
python bench.py --workload pagerank23 --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/b_pr23.json 2>&1
python bench.py --workload pagerank --steps 5 --warmup 3 > gpurun_out/b_pr20.json 2>&1
cat gpurun_out/t.log
