#!/bin/bash
# phase probe of each tools/variants/libtk_*.so and of round 1's package against the current build
mkdir -p gpurun_out
cp paper_2010_10458_b200/libtk.so /tmp/libtk_current.so
for v in /tmp/libtk_current.so tools/variants/libtk_*.so r1; do
  for d in ${SIZES:-25600000}; do
    echo "== $(basename $v) d=$d"
    if [ "$v" = r1 ]; then TK_PKG_PATH=tools/variants/r1 timeout 120 python tools/phase_probe.py $d ${SEL:-mstopk} 2>&1 | tail -1
    else cp $v paper_2010_10458_b200/libtk.so; timeout 120 python tools/phase_probe.py $d ${SEL:-mstopk} 2>&1 | tail -1; fi
  done
done
cp /tmp/libtk_current.so paper_2010_10458_b200/libtk.so
