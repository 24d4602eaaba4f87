#!/bin/bash
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
tag=$1
timeout 900 python -m pytest -m gpu -q -x tests/test_gpu_parity.py -k "generic or golden or engine or both or bulk or fixpoint or zero or nan or selective or throwing or in_scatter or semiring" > gpurun_out/${tag}_tests.log 2>&1; echo "rc=$?" >> gpurun_out/${tag}_tests.log
timeout 600 python tools/generic_bench.py 20 > gpurun_out/${tag}_generic20.log 2>&1
timeout 900 python tools/generic_bench.py 23 > gpurun_out/${tag}_generic23.log 2>&1
tail -3 gpurun_out/${tag}_tests.log; cat gpurun_out/${tag}_generic20.log gpurun_out/${tag}_generic23.log | tail -12
