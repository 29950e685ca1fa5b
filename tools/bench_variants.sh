#!/bin/bash
# bench.py (short) for the current build and every tools/variants/libtk_*.so
cp paper_2010_10458_b200/libtk.so /tmp/libtk_current.so
for v in /tmp/libtk_current.so tools/variants/libtk_*.so; do
  cp $v paper_2010_10458_b200/libtk.so
  for rep in 1 2; do
    timeout 300 python bench.py --steps 40 --warmup 5 --no-cpu-baseline --no-e2e 2>/dev/null | python -c "
import json,sys; l=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('$(basename $v)', round(l['ms_per_step']*1e3,2), {k: round(v['ms_per_launch']*1e3,1) for k,v in l['stages'].items()})"
  done
done
cp /tmp/libtk_current.so paper_2010_10458_b200/libtk.so
