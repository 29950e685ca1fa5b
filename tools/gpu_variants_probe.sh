#!/bin/bash
# launch_probe (C2 EF, C1 no-EF) for the current build and every tools/variants/libtk_*.so; trace_probe for
# the trace variants.  Output: gpurun_out/${TAG}_*.txt
mkdir -p gpurun_out
TAG=${TAG:-vp}
cp paper_2010_10458_b200/libtk.so /tmp/libtk_current.so
for v in /tmp/libtk_current.so tools/variants/libtk_*.so; do
  name=$(basename $v .so)
  cp $v paper_2010_10458_b200/libtk.so
  case $name in
    *trace*)
      timeout 200 python tools/trace_probe.py 25600000 > gpurun_out/${TAG}_${name}_c2.txt 2>&1
      EF=0 timeout 200 python tools/trace_probe.py 1000000 > gpurun_out/${TAG}_${name}_c1.txt 2>&1 ;;
    *)
      for rep in 1 2; do
        echo "== $name rep $rep" >> gpurun_out/${TAG}_launch.txt
        timeout 200 python tools/launch_probe.py 25600000 >> gpurun_out/${TAG}_launch.txt 2>&1
        EF=0 timeout 200 python tools/launch_probe.py 1000000 >> gpurun_out/${TAG}_launch.txt 2>&1
      done ;;
  esac
done
cp /tmp/libtk_current.so paper_2010_10458_b200/libtk.so
