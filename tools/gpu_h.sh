# HiTopK bench reproducibility: dense 2x2 and sparse 1x4, EF-pass compaction on / off
for E in 1 0; do
for CFG in "2 dense" "4 sparse"; do
  set -- $CFG
  TK_EF_COMPACT=$E timeout 150 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port $((29700 + RANDOM % 200)) bench.py --gpus 4 --steps 50 --warmup 5 --group-size $1 --step4 $2 --no-e2e > gpurun_out/hb_${E}_$1$2.json 2> gpurun_out/hb_${E}_$1$2.err
  echo "ef=$E n=$1 step4=$2 rc=$?"
done
done
