#!/bin/bash
# ncu evidence for profiles/: launch list of the bench command (device time per launch) and one
# --set full capture each of k_compress and k_decompress (bench regime, after warm-up), digested
mkdir -p gpurun_out
CMD="python bench.py --ncu --steps 4 --warmup 6"
$CMD > gpurun_out/prof_plain.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/prof_launches.csv $CMD > gpurun_out/prof_launch.log 2>&1; echo "launches rc=$?"
T="python tools/ncu_target.py 25600000 24"
$T > gpurun_out/prof_target_plain.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:k_compress -s 20 -c 1 -o gpurun_out/prof_compress $T > gpurun_out/prof_compress.log 2>&1; echo "compress rc=$?"
python tools/ncu_digest.py gpurun_out/prof_compress.ncu-rep gpurun_out/prof_compress_digest.txt
ncu --set full --clock-control none --import-source on -k regex:k_decompress -s 20 -c 1 -o /tmp/prof_decompress $T > gpurun_out/prof_decompress.log 2>&1; echo "decompress rc=$?"
python tools/ncu_digest.py /tmp/prof_decompress.ncu-rep gpurun_out/prof_decompress_digest.txt
ls -la gpurun_out/prof_compress.ncu-rep
