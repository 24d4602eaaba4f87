mkdir -p gpurun_out
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 1 --master-addr 127.0.0.1 --master-port 29511 bench.py --gpus 1 --steps 5 --warmup 3 > gpurun_out/r02s_torchrun_bfs28.json 2> gpurun_out/r02s_torchrun_bfs28.err; echo rc=$?
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 1 --master-addr 127.0.0.1 --master-port 29512 bench.py --impl reference --gpus 1 --steps 2 --warmup 1 > gpurun_out/r02s_torchrun_ref.json 2> gpurun_out/r02s_torchrun_ref.err; echo rc=$?
timeout 900 python bench.py --sharded --no-cpu-baseline > gpurun_out/r02s_sharded_bfs28.json 2> gpurun_out/r02s_sharded_bfs28.err; echo rc=$?
timeout 900 python bench.py --sharded --workload pagerank28 --no-cpu-baseline > gpurun_out/r02s_sharded_pr28.json 2> gpurun_out/r02s_sharded_pr28.err; echo rc=$?
for f in gpurun_out/r02s_*.json; do echo == $f; tail -1 $f | cut -c1-300; done
for f in gpurun_out/r02s_*.err; do tail -n 3 $f; done
