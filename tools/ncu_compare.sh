#!/bin/bash
# full ncu capture of k_compress (bench regime, 1 launch after 20) for the current build and round 1, digested
mkdir -p gpurun_out
python tools/ncu_target.py > gpurun_out/ncu_cur_plain.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:k_compress -s 20 -c 1 -o /tmp/prof_cur python tools/ncu_target.py > gpurun_out/ncu_cur.log 2>&1; echo "cur rc=$?"
python tools/ncu_digest.py /tmp/prof_cur.ncu-rep gpurun_out/ncu_cur_digest.txt
if [ -z "$NO_R1" ]; then
TK_PKG_PATH=tools/variants/r1 python tools/ncu_target.py > gpurun_out/ncu_r1_plain.log 2>&1 && \
TK_PKG_PATH=tools/variants/r1 ncu --set full --clock-control none --import-source on -k regex:k_compress -s 20 -c 1 -o /tmp/prof_r1 python tools/ncu_target.py > gpurun_out/ncu_r1.log 2>&1; echo "r1 rc=$?"
python tools/ncu_digest.py /tmp/prof_r1.ncu-rep gpurun_out/ncu_r1_digest.txt
fi
