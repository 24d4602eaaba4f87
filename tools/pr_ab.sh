#!/bin/bash
# A/B of the PageRank SpMV kernels (hub vs CTA tiles) at scales 20 and 23.
python -m pytest tests -m gpu -x -q -k "pagerank" 2>&1 | tail -3
python bench.py --workload pagerank23 --steps 5 > gpurun_out/pr23_hub.json 2>&1
GM_PR_HUB=0 python bench.py --workload pagerank23 --steps 5 > gpurun_out/pr23_cta.json 2>&1
python bench.py --workload pagerank --steps 5 > gpurun_out/pr20_hub.json 2>&1
for f in gpurun_out/pr2*.json; do
  python -c "import json,sys; d=json.loads(open(sys.argv[1]).read().strip().splitlines()[-1]); print(sys.argv[1], d['value'], d['roofline']['launch_us'], d['roofline']['frac'], d['e2e']['value'])" $f || tail -5 $f
done
