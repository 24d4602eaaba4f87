mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_rows_f.py -q -x 2>&1 | tail -25 > gpurun_out/tf.log
cat gpurun_out/tf.log
