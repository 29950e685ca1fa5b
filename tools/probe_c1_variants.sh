#!/bin/bash
cp paper_2010_10458_b200/libtk.so /tmp/libtk_current.so
for v in /tmp/libtk_current.so tools/variants/libtk_*.so; do
  cp $v paper_2010_10458_b200/libtk.so; echo "== $(basename $v)"; python tools/c1_probe.py 1000000; python tools/c1_probe.py 4000000
done
cp /tmp/libtk_current.so paper_2010_10458_b200/libtk.so
