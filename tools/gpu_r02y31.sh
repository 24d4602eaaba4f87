#!/bin/bash
# PageRank: hub path at every size -- PR tests (incl. scale 28 vs fp64 and run-to-run), bench lines,
# DRAM / L2 request counters of k_pr_hub at scale 28
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
T=${1:-y31}
timeout 1500 python -m pytest tests -m gpu -q -x -k "pagerank or smoke" > gpurun_out/${T}_tests.log 2>&1; echo "rc=$?" >> gpurun_out/${T}_tests.log
tail -3 gpurun_out/${T}_tests.log
for w in pagerank28 pagerank23 pagerank; do
  timeout 900 python bench.py --workload $w --no-cpu-baseline > gpurun_out/${T}_$w.json 2> gpurun_out/${T}_$w.err
  python -c "import json; d=json.loads(open('gpurun_out/${T}_$w.json').read().strip().splitlines()[-1]); print('$w', d['value'], d['ms_per_step'], d['roofline']['kernel'], d['roofline']['launch_us'], d['roofline']['frac'], d['clocks'])"
done
M="gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_requests_srcunit_tex.sum,lts__t_sectors_srcunit_tex.sum,l1tex__t_requests_pipe_lsu_mem_global_op_ld.sum"
timeout 1200 ncu --metrics $M --clock-control none -k regex:k_pr_hub -s 2 -c 1 --csv python tools/prof_run.py pagerank --scale 28 --reps 1 > gpurun_out/${T}_pr28_counters.csv 2>&1
grep k_pr_hub gpurun_out/${T}_pr28_counters.csv | awk -F'","' '{print $(NF-2), $NF}'
