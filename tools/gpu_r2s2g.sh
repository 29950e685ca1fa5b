#!/bin/bash
mkdir -p gpurun_out
TAG=s2g bash tools/gpu_variants_probe.sh
timeout 1500 python -m pytest tests -x -q -m gpu > gpurun_out/s2g_pytest.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/s2g_pytest.log
