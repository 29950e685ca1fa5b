#!/bin/bash
# build an experimental libtk variant: tools/build_variant.sh NAME -DFLAG ...  -> tools/variants/libtk_NAME.so
name=$1; shift
mkdir -p tools/variants
NCCL=$(python -c "import nvidia.nccl, os; print(list(nvidia.nccl.__path__)[0])")
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 --fmad=false --split-compile=0 -Xcompiler -fPIC,-O2 \
  -shared -o tools/variants/libtk_$name.so paper_2010_10458_b200/csrc/tk.cu -I include -I $NCCL/include -L $NCCL/lib \
  -l:libnccl.so.2 -Xlinker=-rpath,$NCCL/lib -lcudart "$@"
