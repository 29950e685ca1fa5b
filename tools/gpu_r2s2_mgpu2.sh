#!/bin/bash
# 4-GPU: NVLink step-1 pattern ceiling (nvlbench at n = 2 and 4), C3 at P = 4
mkdir -p gpurun_out
CUDA_VISIBLE_DEVICES=0,1 timeout 300 tools/nvlbench > gpurun_out/m2_nvlbench_n2.txt 2>&1; echo "nvl2 rc=$?"
timeout 300 tools/nvlbench > gpurun_out/m2_nvlbench_n4.txt 2>&1; echo "nvl4 rc=$?"
timeout 900 bash tools/trun.sh 4 --dim 110000000 --steps 50 --warmup 5 > gpurun_out/m2_bench_c3_n4.json 2> gpurun_out/m2_bench_c3_n4.err; echo "c3 rc=$?"
