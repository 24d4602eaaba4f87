#!/bin/bash
# Round-2 closing pass: GPU tests, smoke, the default bench (configs[4] BFS
# scale 28) with its CPU baseline, the reference arm, bench lines of the other
# workloads, the default bench's launch list, and a full ncu capture plus the
# DRAM/L2 counters of k_bfs_coop at scale 28, and a full ncu capture of the CF
# item kernel (k_cf_items_grp, both passes).
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
tag=${1:-r02q}
(free -g; nproc; nvidia-smi --query-gpu=name,memory.total,clocks.max.sm --format=csv) > gpurun_out/${tag}_host.txt 2>&1
timeout 2400 python -m pytest tests -m gpu -q > gpurun_out/${tag}_gpu_tests.log 2>&1; echo "tests rc=$?" >> gpurun_out/${tag}_gpu_tests.log
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/${tag}_smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/${tag}_smoke.log
timeout 1200 python bench.py > gpurun_out/${tag}_bench_bfs28.json 2> gpurun_out/${tag}_bench_bfs28.err
timeout 900 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/${tag}_bench_reference.json 2> gpurun_out/${tag}_bench_reference.err
for w in bfs pagerank pagerank23 pagerank28 sssp cf tc; do
  timeout 900 python bench.py --workload $w --no-cpu-baseline > gpurun_out/${tag}_bench_$w.json 2> gpurun_out/${tag}_bench_$w.err
done
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 3000 --csv \
  --log-file gpurun_out/${tag}_bench_bfs28_launches.csv python bench.py --steps 2 --warmup 1 --no-cpu-baseline \
  > gpurun_out/${tag}_ncu_launch_bfs28.log 2>&1
M="gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_requests_srcunit_tex.sum,lts__t_sectors_srcunit_tex.sum,l1tex__t_requests_pipe_lsu_mem_global_op_ld.sum"
timeout 1200 ncu --metrics $M --clock-control none -k regex:k_bfs_coop -s 1 -c 1 --csv python tools/prof_run.py bfs --scale 28 --reps 2 > gpurun_out/${tag}_bfs28_counters.csv 2>&1
timeout 1200 ncu --set full --import-source on --clock-control none -k regex:k_bfs_coop -s 1 -c 1 -f \
  -o /tmp/${tag}_bfs28_coop python tools/prof_run.py bfs --scale 28 --reps 2 > gpurun_out/${tag}_ncu_bfs28.log 2>&1
ncu -i /tmp/${tag}_bfs28_coop.ncu-rep --page raw --csv > gpurun_out/${tag}_bfs28_coop_raw.csv 2>&1
M2="gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_requests_srcunit_tex.sum"
timeout 900 ncu --metrics $M2 --clock-control none -k regex:k_bfs_output -s 1 -c 2 --csv python tools/prof_run.py bfs --scale 28 --reps 3 > gpurun_out/${tag}_bfs28_output_counters.csv 2>&1
timeout 900 ncu --set full --import-source on --clock-control none -k regex:k_cf_items_grp -s 2 -c 2 -f \
  -o /tmp/${tag}_cf_grp python tools/prof_run.py cf --reps 1 > gpurun_out/${tag}_ncu_cf.log 2>&1
ncu -i /tmp/${tag}_cf_grp.ncu-rep --page raw --csv > gpurun_out/${tag}_cf_grp_raw.csv 2>&1
timeout 900 python tools/generic_bench.py 20 > gpurun_out/${tag}_generic20.log 2>&1
timeout 900 python tools/generic_bench.py 23 > gpurun_out/${tag}_generic23.log 2>&1
tail -3 gpurun_out/${tag}_gpu_tests.log; cat gpurun_out/${tag}_smoke.log
for f in gpurun_out/${tag}_bench_*.json; do echo "== $f"; tail -1 $f | cut -c1-400; done
ls -la gpurun_out/${tag}_*
