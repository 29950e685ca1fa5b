#!/bin/bash
# round-2 session-2 measurement: default bench line (twice), C3 line, smoke, ncu launch list + full captures
mkdir -p gpurun_out
timeout 300 python __graft_entry__.py smoke > gpurun_out/s2i_smoke.log 2>&1; echo "smoke rc=$?"; tail -1 gpurun_out/s2i_smoke.log
for i in 1 2; do timeout 900 python bench.py > gpurun_out/s2i_bench_n1_$i.json 2> gpurun_out/s2i_bench_n1_$i.err; echo "bench $i rc=$?"; done
timeout 900 python bench.py --d 110000000 --steps 50 --warmup 5 --no-extra > gpurun_out/s2i_bench_c3_n1.json 2> gpurun_out/s2i_bench_c3_n1.err; echo "c3 rc=$?"
timeout 600 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/s2i_ref_n1.json 2> gpurun_out/s2i_ref_n1.err; echo "ref rc=$?"
CMD="python bench.py --ncu --steps 4 --warmup 6"
$CMD > gpurun_out/s2i_plain.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/s2i_launches.csv $CMD > gpurun_out/s2i_launch.log 2>&1; echo "launches rc=$?"
T="python tools/ncu_target.py 25600000 24"
$T > gpurun_out/s2i_target_plain.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:k_compress -s 20 -c 1 -o gpurun_out/s2i_compress $T > gpurun_out/s2i_compress.log 2>&1; echo "compress rc=$?"
python tools/ncu_digest.py gpurun_out/s2i_compress.ncu-rep gpurun_out/s2i_compress_digest.txt
python tools/ncu_footprint.py gpurun_out/s2i_compress.ncu-rep k_compress > gpurun_out/s2i_footprint.txt 2>&1
ncu --set full --clock-control none --import-source on -k regex:k_decompress -s 20 -c 1 -o /tmp/s2i_decompress $T > gpurun_out/s2i_decompress.log 2>&1; echo "decompress rc=$?"
python tools/ncu_digest.py /tmp/s2i_decompress.ncu-rep gpurun_out/s2i_decompress_digest.txt
