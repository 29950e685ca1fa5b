# multi-GPU bench lines of the next rows and HiTopKComm (4 GPUs)
run() { tag=$1; shift; timeout 200 python -m torch.distributed.run --nnodes=1 --nproc-per-node $NP --master-addr 127.0.0.1 --master-port $((29700 + RANDOM % 250)) bench.py --gpus $NP --steps 100 --warmup 10 --no-e2e "$@" > gpurun_out/mv_$tag.json 2> gpurun_out/mv_$tag.err; echo "$tag rc=$?"; }
NP=4 run n4_exact --select exact
NP=4 run n4_f16 --wire f16
NP=4 run n4_f16_nccl --wire f16 --ag-mode nccl
NP=4 run n4_sgd --sgd 0.01
NP=4 run h22_dense --group-size 2
NP=4 run h22_sparse --group-size 2 --step4 sparse
NP=4 run h14_sparse --group-size 4 --step4 sparse
