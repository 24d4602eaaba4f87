mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -k "sharded" 2>&1 | tail -15 > gpurun_out/ts.log
cat gpurun_out/ts.log
