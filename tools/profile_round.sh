#!/bin/bash
# Round profile on one B200: GPU tests, bench lines for every workload, the
# reference arm, ncu launch lists of the bench steps, and one ncu --set full
# capture per hot kernel.  Usage: tools/profile_round.sh <tag>
tag=${1:-rXX}
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
python -m pytest tests -m gpu -x -q > gpurun_out/${tag}_gpu_tests.log 2>&1; echo "tests rc=$?" >> gpurun_out/${tag}_gpu_tests.log
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/${tag}_smoke.log 2>&1
for w in bfs pagerank pagerank23 sssp cf tc; do
  timeout 900 python bench.py --workload $w > gpurun_out/${tag}_bench_$w.json 2> gpurun_out/${tag}_bench_$w.err
done
timeout 900 python bench.py --impl reference > gpurun_out/${tag}_bench_reference.json 2> gpurun_out/${tag}_bench_reference.err
for w in bfs sssp cf pagerank23; do
  timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 2000 --csv \
    --log-file gpurun_out/${tag}_bench_${w}_launches.csv python bench.py --workload $w --steps 2 --warmup 1 --no-cpu-baseline \
    > gpurun_out/${tag}_ncu_launch_$w.log 2>&1
done
timeout 600 ncu --set full --import-source on --clock-control none -k regex:k_bfs_coop -s 1 -c 1 \
  -o gpurun_out/${tag}_bfs23_coop python tools/prof_run.py bfs --reps 2 > gpurun_out/${tag}_ncu_bfs.log 2>&1
timeout 600 ncu --set full --import-source on --clock-control none -k regex:"^k_sssp_pull$" -s 3 -c 1 \
  -o gpurun_out/${tag}_sssp23_pull python tools/prof_run.py sssp --reps 1 > gpurun_out/${tag}_ncu_sssp.log 2>&1
timeout 600 ncu --set full --import-source on --clock-control none -k regex:k_cf_items -c 2 \
  -o gpurun_out/${tag}_cf_items python tools/prof_run.py cf --reps 1 > gpurun_out/${tag}_ncu_cf.log 2>&1
tail -1 gpurun_out/${tag}_gpu_tests.log; cat gpurun_out/${tag}_smoke.log
for w in bfs pagerank pagerank23 sssp cf tc reference; do
  python -c "import json,sys; d=json.loads(open(sys.argv[1]).read().strip().splitlines()[-1]); print(sys.argv[1], d.get('value'), d.get('ms_per_step'), (d.get('roofline') or {}).get('frac'), (d.get('e2e') or {}).get('value'))" gpurun_out/${tag}_bench_$w.json || tail -3 gpurun_out/${tag}_bench_$w.err
done
ls gpurun_out/${tag}_*.ncu-rep
