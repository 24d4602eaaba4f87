#!/bin/bash
# r02 profile pass: L2 request rate microbenchmark + per-kernel request / DRAM
# counters of the dominant kernels (read back with tools/summarize_ncu.py).
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
tag=r02s
M="gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_requests_srcunit_tex.sum,lts__t_sectors_srcunit_tex.sum,lts__t_sectors_srcunit_tex_lookup_hit.sum,l1tex__t_requests_pipe_lsu_mem_global_op_ld.sum,l1tex__t_sectors_pipe_lsu_mem_global_op_ld.sum"
./tools/gather_bench > gpurun_out/${tag}_gather_bench.txt 2>&1
timeout 900 ncu --metrics $M --clock-control none -k regex:k_pr_hub -s 1 -c 1 --csv python tools/prof_run.py pagerank --scale 23 --reps 1 > gpurun_out/${tag}_pr23_hub.csv 2>&1
timeout 900 ncu --metrics $M --clock-control none -k regex:k_bfs_coop -s 1 -c 1 --csv python tools/prof_run.py bfs --scale 23 --reps 2 > gpurun_out/${tag}_bfs23.csv 2>&1
timeout 1200 ncu --metrics $M --clock-control none -k regex:k_bfs_coop -s 1 -c 1 --csv python tools/prof_run.py bfs --scale 28 --reps 2 > gpurun_out/${tag}_bfs28.csv 2>&1
timeout 1200 ncu --metrics $M --clock-control none -k regex:k_pr_spmv -s 1 -c 1 --csv python tools/prof_run.py pagerank --scale 28 --reps 1 > gpurun_out/${tag}_pr28_spmv.csv 2>&1
timeout 900 ncu --metrics $M --clock-control none -k regex:k_cf_items -c 2 --csv python tools/prof_run.py cf --reps 1 > gpurun_out/${tag}_cf.csv 2>&1
cat gpurun_out/${tag}_gather_bench.txt | head -20
for f in gpurun_out/${tag}_*.csv; do echo "== $f"; grep -E '"(gpu__time|dram__|lts__|l1tex__)' $f | awk -F'","' '{print $(NF-2), $(NF)}' | head -20; done
