#!/bin/bash
# 4-GPU pass: HiTopKComm soak (50 rounds of fresh contexts), multi-GPU parity tests, bench lines
mkdir -p gpurun_out
timeout 1200 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29611 \
  tools/hitopk_soak.py 50 100 > gpurun_out/m_soak.txt 2> gpurun_out/m_soak.err; echo "soak rc=$?"; tail -2 gpurun_out/m_soak.txt
timeout 1800 python -m pytest -q -m gpu tests/test_multigpu.py > gpurun_out/m_pytest.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/m_pytest.log
run() { name=$1; shift; timeout 600 "$@" > gpurun_out/m_bench_$name.json 2> gpurun_out/m_bench_$name.err; echo "bench $name rc=$?"; }
run n2 bash tools/trun.sh 2
run n4 bash tools/trun.sh 4
run c3_n4 bash tools/trun.sh 4 --d 110000000 --steps 50 --warmup 5
run h22_dense bash tools/trun.sh 4 --group-size 2 --steps 50 --warmup 5 --no-e2e
run h22_sparse bash tools/trun.sh 4 --group-size 2 --step4 sparse --steps 50 --warmup 5 --no-e2e
run h14_dense bash tools/trun.sh 4 --group-size 4 --steps 50 --warmup 5 --no-e2e
run h14_sparse bash tools/trun.sh 4 --group-size 4 --step4 sparse --steps 50 --warmup 5 --no-e2e
run h22_dense_r1e2 bash tools/trun.sh 4 --group-size 2 --rho 0.01 --steps 50 --warmup 5 --no-e2e
run h14_sparse_r1e2 bash tools/trun.sh 4 --group-size 4 --rho 0.01 --step4 sparse --steps 50 --warmup 5 --no-e2e
run ref_n4 bash tools/trun.sh 4 --impl reference --steps 3 --warmup 3
