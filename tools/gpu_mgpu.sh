set -x
timeout 1200 python -m pytest tests/test_multigpu.py -x -q > gpurun_out/mgpu_tests.log 2>&1; echo "mgpu tests rc=$?"; tail -3 gpurun_out/mgpu_tests.log
for N in 2 4; do
  timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 2950$N bench.py --gpus $N --steps 100 --warmup 10 > gpurun_out/bench_n$N.json 2> gpurun_out/bench_n$N.err; echo "bench n=$N rc=$?"
  timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 2951$N bench.py --gpus $N --steps 100 --warmup 10 --ag-mode nccl --no-e2e > gpurun_out/bench_n${N}_nccl.json 2> gpurun_out/bench_n${N}_nccl.err; echo "bench nccl n=$N rc=$?"
done
timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29520 bench.py --gpus 4 --steps 50 --warmup 5 --group-size 2 --no-e2e > gpurun_out/bench_h22.json 2> gpurun_out/bench_h22.err; echo "bench hitopk rc=$?"
timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29521 bench.py --gpus 4 --steps 50 --warmup 5 --group-size 4 --step4 sparse --no-e2e > gpurun_out/bench_h14s.json 2> gpurun_out/bench_h14s.err; echo "bench hitopk14s rc=$?"
