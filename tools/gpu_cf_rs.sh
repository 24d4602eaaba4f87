#!/bin/bash
# CF reduce-scatter kernel variants (GM_CF_G=50/51/52) against the shipped G=5.
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
tag=${1:-r02q_cf}
for G in 5 50 51 52; do GM_CF_G=$G timeout 600 python tools/cf_exp.py >> gpurun_out/${tag}.txt 2>&1; done
GM_CF_G=51 timeout 900 python -m pytest tests -m gpu -q -k "cf" > gpurun_out/${tag}_tests51.log 2>&1; echo "rc=$?" >> gpurun_out/${tag}_tests51.log
cat gpurun_out/${tag}.txt; tail -3 gpurun_out/${tag}_tests51.log
