mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_configs.py -q -x -k "cf" 2>&1 | tail -3 > gpurun_out/tcf.log
timeout 900 python bench.py --workload cf --steps 3 --warmup 3 > gpurun_out/b_cf.json 2> gpurun_out/b_cf.err
cat gpurun_out/tcf.log; tail -n 3 gpurun_out/b_cf.err
