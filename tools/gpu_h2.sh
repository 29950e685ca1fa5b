# HiTopK 1x4 sparse crash hunt: 3 runs each of default / NVLS off / NCCL reduce-scatter
run() { tag=$1; shift; for i in 1 2 3; do env "$@" timeout 120 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port $((29700 + RANDOM % 250)) bench.py --gpus 4 --steps 50 --warmup 5 --group-size 4 --step4 sparse --no-e2e --no-cpu-baseline $EXTRA > /dev/null 2> gpurun_out/h2_${tag}_$i.err; echo "$tag run $i rc=$?"; done; }
EXTRA="" run default TK_EF_COMPACT=1
EXTRA="" run nonvls TK_EF_COMPACT=1 NCCL_NVLS_ENABLE=0
EXTRA="--rs-mode nccl" run rsnccl TK_EF_COMPACT=1
