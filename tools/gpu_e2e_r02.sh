cd "$(dirname "$0")" 2>/dev/null; cd /root/repo
tag=r02qe
timeout 900 python -m pytest tests -m gpu -q -k "host_async" > gpurun_out/${tag}_tests.log 2>&1; echo "rc=$?" >> gpurun_out/${tag}_tests.log
timeout 900 python tools/pr28_e2e.py 28 > gpurun_out/${tag}_pr28_e2e.txt 2>&1
for w in pagerank28 pagerank sssp; do
  timeout 900 python bench.py --workload $w --no-cpu-baseline > gpurun_out/${tag}_bench_$w.json 2> gpurun_out/${tag}_bench_$w.err
done
tail -3 gpurun_out/${tag}_tests.log; cat gpurun_out/${tag}_pr28_e2e.txt
for f in gpurun_out/${tag}_bench_*.json; do tail -1 $f | cut -c1-200; done
