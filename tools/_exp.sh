mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_rows_f.py -q -x 2>&1 | tail -5 > gpurun_out/tf.log
timeout 900 python bench.py --workload tc --steps 5 --warmup 3 > gpurun_out/b_tc.json 2> gpurun_out/b_tc.err
timeout 600 python bench.py --workload tc --scale 23 --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/b_tc23.json 2> gpurun_out/b_tc23.err
cat gpurun_out/tf.log
