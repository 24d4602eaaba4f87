#!/bin/bash
# quick GPU check: the named pytest selection, output to gpurun_out/<tag>_*.log
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
tag=$1; shift
timeout ${GM_TIMEOUT:-1200} python -m pytest "$@" > gpurun_out/${tag}_tests.log 2>&1; echo "rc=$?" >> gpurun_out/${tag}_tests.log
tail -40 gpurun_out/${tag}_tests.log
