mkdir -p gpurun_out
timeout 300 python -m pytest tests -m gpu -q -x -k "pagerank" 2>&1 | tail -2 > gpurun_out/t.log
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:k_pr_spmv -c 6 --csv --log-file gpurun_out/hh_default.csv python tools/pr_once.py 23 > /dev/null 2>&1
for v in hot2k hot4k hot8k hot16k; do
  L="GM_LIB=_variants/$v/libgraphmat_b200.so"
  env $L timeout 300 python -m pytest tests -m gpu -q -x -k "pagerank" 2>&1 | tail -1 >> gpurun_out/t.log
  env $L timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:k_pr_spmv -c 6 --csv --log-file gpurun_out/hh_${v}.csv python tools/pr_once.py 23 > /dev/null 2>&1
done
cat gpurun_out/t.log
