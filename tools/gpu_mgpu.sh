#!/bin/bash
# multi-GPU pass (run with gpurun --gpus 4): multi-GPU parity tests, benches at P = 2 / 4 (flat and
# HiTopKComm), and a soak of the HiTopKComm peer-sum kernel with the EF-pass compaction
mkdir -p gpurun_out
NG=$(nvidia-smi -L | wc -l)
timeout 1500 python -m pytest -q -m gpu tests/test_multigpu.py ${PYT_K:+-k "$PYT_K"} > gpurun_out/pytest_mgpu.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/pytest_mgpu.log
run() { name=$1; shift; timeout 600 "$@" > gpurun_out/bench_$name.json 2> gpurun_out/bench_$name.err; echo "bench $name rc=$?"; }
[ -z "$NO_BENCH" ] && {
run n2 bash tools/trun.sh 2 --steps 30 --warmup 5 --no-e2e
run n4 bash tools/trun.sh 4 --steps 30 --warmup 5 --no-e2e
run h22_dense bash tools/trun.sh 4 --group-size 2 --steps 30 --warmup 5 --no-e2e
run h22_sparse bash tools/trun.sh 4 --group-size 2 --step4 sparse --steps 30 --warmup 5 --no-e2e
run h14_dense bash tools/trun.sh 4 --group-size 4 --steps 30 --warmup 5 --no-e2e
run h14_sparse bash tools/trun.sh 4 --group-size 4 --step4 sparse --steps 30 --warmup 5 --no-e2e
run h22_dense_r1e2 bash tools/trun.sh 4 --group-size 2 --rho 0.01 --steps 30 --warmup 5 --no-e2e
run h14_sparse_r1e2 bash tools/trun.sh 4 --group-size 4 --rho 0.01 --step4 sparse --steps 30 --warmup 5 --no-e2e
}
[ -n "$SOAK" ] && for i in $(seq 1 $SOAK); do
  timeout 300 bash tools/trun.sh 4 --group-size 4 --step4 sparse --steps 100 --warmup 5 --no-e2e --no-cpu-baseline > gpurun_out/soak_$i.json 2> gpurun_out/soak_$i.err; echo "soak 1x4 sparse $i rc=$?"
  timeout 300 bash tools/trun.sh 4 --group-size 2 --steps 100 --warmup 5 --no-e2e --no-cpu-baseline > gpurun_out/soak2_$i.json 2> gpurun_out/soak2_$i.err; echo "soak 2x2 dense $i rc=$?"
done
true
