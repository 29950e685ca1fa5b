#!/bin/bash
# round-2 session-2 first call: state check (GPU suite, smoke, bench), phase probe, EF-pattern ceiling
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/s2_smi.txt
timeout 300 tools/efbench > gpurun_out/s2_efbench.txt 2>&1; echo "efbench rc=$?"
timeout 300 python tools/phase_probe.py 25600000 > gpurun_out/s2_phase.txt 2>&1; echo "phase rc=$?"
timeout 300 python tools/phase_probe.py 1000000 >> gpurun_out/s2_phase.txt 2>&1
timeout 600 python bench.py --steps 50 --warmup 5 > gpurun_out/s2_bench.json 2> gpurun_out/s2_bench.err; echo "bench rc=$?"
timeout 1500 python -m pytest tests -x -q -m gpu > gpurun_out/s2_pytest.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/s2_pytest.log
