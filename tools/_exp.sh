mkdir -p gpurun_out/prof
P=gpurun_out/prof
NCU="timeout 900 ncu --set full --import-source on --clock-control none"
$NCU -k regex:k_pr_spmv --launch-skip 2 -c 1 -o $P/r01_pr23_spmv python tools/prof_run.py pagerank --scale 23 > $P/l1.log 2>&1
$NCU -k regex:k_pr_spmv --launch-skip 2 -c 1 -o $P/r01_pr20_spmv python tools/prof_run.py pagerank --scale 20 > $P/l2.log 2>&1
$NCU -k regex:k_bfs_coop --launch-skip 1 -c 1 -o $P/r01_bfs23_coop python tools/prof_run.py bfs --scale 23 > $P/l3.log 2>&1
$NCU -k regex:k_sssp_push --launch-skip 6 -c 1 -o $P/r01_sssp23_push python tools/prof_run.py sssp --scale 23 > $P/l4.log 2>&1
$NCU -k regex:k_cf_items --launch-skip 2 -c 1 -o $P/r01_cf_items python tools/prof_run.py cf > $P/l5.log 2>&1
$NCU -k regex:k_pr_spmv --launch-skip 1 -c 1 -o $P/r01_pr28_spmv python tools/prof_run.py pagerank --scale 28 --reps 1 > $P/l6.log 2>&1
$NCU -k regex:k_bfs_coop --launch-skip 1 -c 1 -o $P/r01_bfs28_coop python tools/prof_run.py bfs --scale 28 > $P/l7.log 2>&1
for w in bfs pagerank23 sssp cf; do
  timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file $P/r01_bench_${w}_launches.csv python bench.py --workload $w --steps 2 --warmup 1 --no-cpu-baseline > $P/lb_$w.log 2>&1
done
ls -la $P
