mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q -x -k "shard or pagerank" 2>&1 | tail -3 > gpurun_out/ts.log
cat gpurun_out/ts.log
