#!/bin/bash
# GPU test pass: the whole -m gpu suite (no -x: report every failure), then smoke
mkdir -p gpurun_out
timeout ${PYT_TIMEOUT:-1500} python -m pytest tests -q -m gpu ${PYT_ARGS} ${PYT_K:+-k "$PYT_K"} > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"
tail -30 gpurun_out/pytest_gpu.log
timeout 300 python __graft_entry__.py smoke > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?"; tail -2 gpurun_out/smoke.log
