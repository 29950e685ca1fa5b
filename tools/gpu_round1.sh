#!/bin/bash
# smoke + bench + ncu launch list + one full ncu capture of the count pass and the EF pass
set -x
mkdir -p gpurun_out
python __graft_entry__.py smoke > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/smoke.log
python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err; echo "bench rc=$?"
python bench.py --ncu --steps 3 --warmup 3 > gpurun_out/plain_ncu_cmd.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv \
    python bench.py --ncu --steps 3 --warmup 3 > gpurun_out/ncu_launches.log 2>&1; echo "ncu1 rc=$?"
ncu --set full --clock-control none --import-source on -k regex:"k_count|k_ef_stats|k_select|k_decompress" -s 8 -c 8 \
    -o gpurun_out/prof_r1 python bench.py --ncu --steps 2 --warmup 1 > gpurun_out/ncu_full.log 2>&1; echo "ncu2 rc=$?"
