#!/bin/bash
# tools/gpu.sh TASK — the GPU-side command sets run through gpurun (outputs under gpurun_out/), e.g.
#   gpurun --timeout 2400 -- 'bash tools/gpu.sh tests'
#   gpurun --gpus 4 --timeout 3600 -- 'bash tools/gpu.sh mgpu'
# TASK:
#   tests    the whole `pytest -m gpu` suite (no -x: every failure is reported), then smoke()
#   bench    the default bench line (N = 1, C2), the C3 line and the reference arm
#   profile  ncu launch list of the bench command; `--set full` of k_compress / k_decompress in the
#            bench regime, digested (tools/ncu_digest.py), and k_compress's executed-code footprint
#   probes   per-call device time (tools/launch_probe.py) and per-CTA phase timelines
#            (tools/trace_probe.py, needs a -DTK_PHASE_TRACE variant) of the current build and of every
#            tools/variants/libtk_*.so (built with tools/build_variant.sh)
#   sweep    the C5 size / density / N sweep (tools/sweep_c5.py) and the EF-pattern / cold-code
#            microbenchmarks (tools/efbench, tools/icache_bench; nvcc lines in their headers)
#   mgpu     (4 GPUs) multi-GPU parity tests, bench lines at P = 2 / 4 (flat) and HiTopKComm 2x2 / 1x4
#            dense / sparse (rho = 1e-3 and 1e-2), C3 at P = 4, the 100-context HiTopKComm soak and the
#            NVLink ceiling of step 1's access pattern (tools/nvlbench)
#   final    round-end style: tests, smoke and bench lines at N = 1, 2, 4
set -u
mkdir -p gpurun_out
task=${1:-tests}
# (timeout cannot run a shell function: the launcher is a command line)
TORCHRUN="python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1"
case $task in
tests)
  timeout 1800 python -m pytest tests -q -m gpu > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"
  tail -3 gpurun_out/pytest_gpu.log
  timeout 300 python __graft_entry__.py smoke > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?"; tail -1 gpurun_out/smoke.log ;;
bench)
  timeout 900 python bench.py > gpurun_out/bench_n1.json 2> gpurun_out/bench_n1.err; echo "bench rc=$?"
  timeout 900 python bench.py --dim 110000000 --steps 50 --warmup 5 --no-extra > gpurun_out/bench_c3_n1.json 2> gpurun_out/bench_c3_n1.err; echo "c3 rc=$?"
  timeout 600 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/bench_ref_n1.json 2> gpurun_out/bench_ref_n1.err; echo "ref rc=$?" ;;
profile)
  CMD="python bench.py --ncu --steps 4 --warmup 6"
  $CMD > gpurun_out/prof_plain.log 2>&1 && \
  ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/prof_launches.csv $CMD > gpurun_out/prof_launch.log 2>&1
  echo "launches rc=$?"
  T="python tools/ncu_target.py 25600000 24"
  $T > gpurun_out/prof_target_plain.log 2>&1 && \
  ncu --set full --clock-control none --import-source on -k regex:k_compress -s 20 -c 1 -o gpurun_out/prof_compress $T > gpurun_out/prof_compress.log 2>&1
  echo "compress rc=$?"
  python tools/ncu_digest.py gpurun_out/prof_compress.ncu-rep gpurun_out/prof_compress_digest.txt
  python tools/ncu_footprint.py gpurun_out/prof_compress.ncu-rep k_compress 0 gpurun_out/prof_compress_pcs.csv > gpurun_out/prof_footprint.txt 2>&1
  ncu --set full --clock-control none --import-source on -k regex:k_decompress -s 20 -c 1 -o /tmp/prof_decompress $T > gpurun_out/prof_decompress.log 2>&1
  echo "decompress rc=$?"
  python tools/ncu_digest.py /tmp/prof_decompress.ncu-rep gpurun_out/prof_decompress_digest.txt ;;
probes)
  cp paper_2010_10458_b200/libtk.so /tmp/libtk_current.so
  for v in /tmp/libtk_current.so tools/variants/libtk_*.so; do
    [ -f "$v" ] || continue
    name=$(basename $v .so)
    cp $v paper_2010_10458_b200/libtk.so
    case $name in
      *trace*)
        timeout 200 python tools/trace_probe.py 25600000 > gpurun_out/probe_${name}_c2.txt 2>&1
        EF=0 timeout 200 python tools/trace_probe.py 1000000 > gpurun_out/probe_${name}_c1.txt 2>&1 ;;
      *)
        echo "== $name" >> gpurun_out/probe_launch.txt
        timeout 200 python tools/launch_probe.py 25600000 >> gpurun_out/probe_launch.txt 2>&1
        EF=0 timeout 200 python tools/launch_probe.py 1000000 >> gpurun_out/probe_launch.txt 2>&1 ;;
    esac
  done
  cp /tmp/libtk_current.so paper_2010_10458_b200/libtk.so ;;
sweep)
  timeout 2000 python tools/sweep_c5.py gpurun_out/c5_sweep.jsonl > gpurun_out/sweep.log 2>&1; echo "sweep rc=$?"
  [ -x tools/efbench ] && timeout 300 tools/efbench > gpurun_out/efbench.txt 2>&1
  [ -x tools/icache_bench ] && timeout 300 tools/icache_bench > gpurun_out/icache_bench.txt 2>&1
  true ;;
mgpu)
  timeout 1800 python -m pytest -q -m gpu tests/test_multigpu.py > gpurun_out/pytest_mgpu.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/pytest_mgpu.log
  run() { name=$1; shift; timeout 600 "$@" > gpurun_out/mbench_$name.json 2> gpurun_out/mbench_$name.err; echo "bench $name rc=$?"; }
  run n2 bash tools/trun.sh 2
  run n4 bash tools/trun.sh 4
  run c3_n4 bash tools/trun.sh 4 --dim 110000000 --steps 50 --warmup 5
  for cfg in "h22_dense --group-size 2" "h22_sparse --group-size 2 --step4 sparse" "h14_dense --group-size 4" \
             "h14_sparse --group-size 4 --step4 sparse" "h22_dense_r1e2 --group-size 2 --rho 0.01" \
             "h14_sparse_r1e2 --group-size 4 --rho 0.01 --step4 sparse"; do
    set -- $cfg; name=$1; shift
    run $name bash tools/trun.sh 4 --steps 50 --warmup 5 --no-e2e "$@"
  done
  timeout 1200 $TORCHRUN --nproc-per-node 4 --master-port 29611 tools/hitopk_soak.py 50 100 \
    > gpurun_out/hitopk_soak.txt 2> gpurun_out/hitopk_soak.err; echo "soak rc=$?"
  [ -x tools/nvlbench ] && { CUDA_VISIBLE_DEVICES=0,1 timeout 300 tools/nvlbench > gpurun_out/nvlbench_n2.txt 2>&1;
                             timeout 300 tools/nvlbench > gpurun_out/nvlbench_n4.txt 2>&1; }
  true ;;
final)
  bash tools/gpu.sh tests
  timeout 900 python bench.py > gpurun_out/final_n1.json 2> gpurun_out/final_n1.err; echo "bench n1 rc=$?"
  NG=$(nvidia-smi -L | wc -l)
  for N in 2 4; do
    [ $NG -ge $N ] || continue
    timeout 600 bash tools/trun.sh $N > gpurun_out/final_n$N.json 2> gpurun_out/final_n$N.err; echo "bench n$N rc=$?"
  done ;;
*) echo "unknown task $task"; exit 2 ;;
esac
