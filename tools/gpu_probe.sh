#!/bin/bash
# per-phase device time of k_compress (bench regime) at several sizes + grid-barrier cost
mkdir -p gpurun_out
for d in 25600000 1000000 110000000; do
  timeout 300 python tools/phase_probe.py $d mstopk >> gpurun_out/phase_probe.log 2>&1
done
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/bb tools/barrier_bench.cu && timeout 120 /tmp/bb >> gpurun_out/barrier_bench.log 2>&1
nproc > gpurun_out/host.txt; lscpu | grep -i "model name" >> gpurun_out/host.txt; free -g >> gpurun_out/host.txt
