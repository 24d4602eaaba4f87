mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_rows_f.py tests/test_abi.py -q -x 2>&1 | tail -30 > gpurun_out/tf.log
cat gpurun_out/tf.log
