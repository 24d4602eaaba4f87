#!/bin/bash
# PageRank scale-23 superstep: hub kernel alone vs hub + propagation-blocked tail.
cd "$(dirname "$0")/.."
GM_PR_PB=0 GM_SAVE=gpurun_out/pr23_hub.npy timeout 300 python tools/pr_exp.py 23
for cfg in "GM_PB_ROUNDS=1" "GM_PB_ROUNDS=2" "GM_PB_ROUNDS=1 GM_PB_CAP=32768 GM_PB_BIG=32768" "GM_PB_ROUNDS=1 GM_PB_CW=49152"; do
  env GM_PR_PB=1 GM_CMP=gpurun_out/pr23_hub.npy $cfg timeout 300 python tools/pr_exp.py 23 || echo "FAILED $cfg"
done
GM_PR_PB=1 timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sector_hit_rate.pct,sm__warps_active.avg.pct_of_peak_sustained_active --clock-control none -k regex:"k_pb_scatter|k_pb_bucket|k_pr_hub" --launch-skip 30 -c 3 --csv python tools/pr_exp.py 23 > gpurun_out/pb_ncu.csv 2>gpurun_out/pb_ncu.err
grep -v "^==\|^{" gpurun_out/pb_ncu.csv | python -c "
import csv,sys
rows={}
for r in csv.DictReader(sys.stdin):
    k=(int(r['ID']), r['Kernel Name'][11:30], r['Grid Size'])
    rows.setdefault(k,{})[r['Metric Name']]=r['Metric Value']
for k,v in sorted(rows.items()): print(k, v)
"
