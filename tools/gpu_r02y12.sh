#!/bin/bash
# generic engine: hub-row kernel tests + superstep timings
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
T=${1:-y12}
timeout 900 python -m pytest -m gpu -q -x tests/test_gpu_parity.py -k "generic or golden or engine or both or bulk or fixpoint or zero or nan or selective or throwing or in_scatter or semiring or callback or relabel_invariance" > gpurun_out/${T}_tests.log 2>&1; echo "rc=$?" >> gpurun_out/${T}_tests.log
tail -15 gpurun_out/${T}_tests.log
timeout 600 python tools/generic_bench.py 20 > gpurun_out/${T}_generic20.log 2>&1
timeout 900 python tools/generic_bench.py 23 > gpurun_out/${T}_generic23.log 2>&1
cat gpurun_out/${T}_generic20.log gpurun_out/${T}_generic23.log | tail -12
