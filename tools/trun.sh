#!/bin/bash
# tools/trun.sh NGPU [bench.py args...]: bench.py under torchrun on NGPU local GPUs (127.0.0.1 rendezvous)
n=$1; shift
exec python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 --master-port $((29500 + RANDOM % 1000)) bench.py --gpus $n "$@"
