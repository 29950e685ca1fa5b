mkdir -p gpurun_out
S=/usr/local/cuda/bin/compute-sanitizer
for tool in memcheck racecheck synccheck initcheck; do
  timeout 300 $S --tool $tool --error-exitcode 7 python tools/sanitize_step.py > gpurun_out/san_$tool.log 2>&1; echo "$tool rc=$?"; tail -2 gpurun_out/san_$tool.log
done
timeout 300 $S --tool memcheck --error-exitcode 7 python tools/sanitize_step.py --select exact --wire f16 --sgd > gpurun_out/san_memcheck_exact.log 2>&1; echo "memcheck exact rc=$?"; tail -2 gpurun_out/san_memcheck_exact.log
