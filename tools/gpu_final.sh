# round-end style validation: every GPU test (1-4 GPUs), smoke, and bench lines at N=1,2,4
mkdir -p gpurun_out
timeout 1800 python -m pytest tests -x -q -m gpu > gpurun_out/final_pytest.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/final_pytest.log
python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/final_smoke.log 2>&1; echo "smoke rc=$?"
python bench.py > gpurun_out/final_n1.json 2> gpurun_out/final_n1.err; echo "bench n1 rc=$?"
for N in 2 4; do
  timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port $((29600 + N)) bench.py --gpus $N > gpurun_out/final_n$N.json 2> gpurun_out/final_n$N.err; echo "bench n$N rc=$?"
done
timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29655 bench.py --impl reference --gpus 2 --steps 3 --warmup 3 > gpurun_out/final_ref_n2.json 2> gpurun_out/final_ref_n2.err; echo "ref n2 rc=$?"
