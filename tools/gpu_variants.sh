# bench lines for the NEXT rows (exact selector F1, FP16 wire F3, fused SGD update F4) at N=1
mkdir -p gpurun_out
python bench.py --steps 100 --warmup 10 --no-e2e --no-cpu-baseline --select exact > gpurun_out/v_exact.json 2> gpurun_out/v_exact.err; echo "exact rc=$?"
python bench.py --steps 100 --warmup 10 --no-e2e --no-cpu-baseline --wire f16 > gpurun_out/v_f16.json 2> gpurun_out/v_f16.err; echo "f16 rc=$?"
python bench.py --steps 100 --warmup 10 --no-e2e --no-cpu-baseline --sgd 0.01 > gpurun_out/v_sgd.json 2> gpurun_out/v_sgd.err; echo "sgd rc=$?"
python bench.py --steps 50 --warmup 5 --no-e2e --no-cpu-baseline --d 110000000 > gpurun_out/v_c3.json 2> gpurun_out/v_c3.err; echo "c3 rc=$?"
python bench.py --steps 100 --warmup 10 --no-e2e --no-cpu-baseline --d 1000000 > gpurun_out/v_c1.json 2> gpurun_out/v_c1.err; echo "c1 rc=$?"
python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/v_ref.json 2> gpurun_out/v_ref.err; echo "ref rc=$?"
