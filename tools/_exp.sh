mkdir -p gpurun_out
timeout 900 python tools/diag28.py 28 2>&1 | grep -v Assertion | head -20 > gpurun_out/diag28.txt
SECONDS=0
timeout 1500 python -m pytest tests/test_gpu_scale28.py -x -q > gpurun_out/t28.log 2>&1
echo "rc=$? secs=$SECONDS" >> gpurun_out/t28.log
timeout 600 python bench.py --workload bfs28 --steps 5 --warmup 3 > gpurun_out/b_bfs28.json 2> gpurun_out/b_bfs28.err
timeout 600 python bench.py --workload pagerank28 --steps 2 --warmup 3 > gpurun_out/b_pr28.json 2> gpurun_out/b_pr28.err
cat gpurun_out/diag28.txt; tail -4 gpurun_out/t28.log
