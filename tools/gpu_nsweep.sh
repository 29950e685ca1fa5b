#!/bin/bash
# N (number of samplings, Alg. 1) sweep at C2 on one GPU: SURVEY F3's N = 30 and C5's {5, 10, 20}
mkdir -p gpurun_out
for N in 5 20 30; do
  python bench.py --n-iters $N --no-cpu-baseline > gpurun_out/bench_n$N.json 2> gpurun_out/bench_n$N.err; echo "N=$N rc=$?"
done
