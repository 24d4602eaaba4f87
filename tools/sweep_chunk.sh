for c in 1 2 4 8 16 32; do
  echo "chunk $c: $(GM_BFS_PULL_CHUNK=$c timeout 300 python bench.py --workload bfs --steps 20 --warmup 5 --no-cpu-baseline 2>/dev/null | python -c 'import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print(d["value"], d["ms_per_step"], [s["us"] for s in d["per_superstep"]])')"
done
for c in 8 16 32; do
  echo "28 chunk $c: $(GM_BFS_PULL_CHUNK=$c timeout 300 python bench.py --steps 5 --warmup 3 --no-cpu-baseline 2>/dev/null | python -c 'import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print(d["value"], d["ms_per_step"], [s["us"] for s in d["per_superstep"]])')"
done
