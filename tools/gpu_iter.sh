#!/bin/bash
# quick iteration: parity tests, smoke, bench, launch list (+ optional full ncu capture of a kernel regex)
mkdir -p gpurun_out
timeout 900 python -m pytest tests -x -q -m gpu > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"
tail -3 gpurun_out/pytest_gpu.log
python __graft_entry__.py smoke > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?"
python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err; echo "bench rc=$?"
python bench.py --ncu --steps 3 --warmup 3 > gpurun_out/plain_ncu_cmd.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv \
    python bench.py --ncu --steps 3 --warmup 3 > gpurun_out/ncu_launches.log 2>&1; echo "ncu launches rc=$?"
if [ -n "$NCU_REGEX" ]; then
ncu --set full --clock-control none --import-source on -k regex:"$NCU_REGEX" -s ${NCU_SKIP:-6} -c ${NCU_COUNT:-6} \
    -o gpurun_out/prof python bench.py --ncu --steps 2 --warmup 1 > gpurun_out/ncu_full.log 2>&1; echo "ncu full rc=$?"
fi
