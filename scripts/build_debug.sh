#!/bin/bash
# debug build with device printf -> paper_1606_05973_b200/libccl_b200_dbg.so
set -e
cd "$(dirname "$0")/.."
NCCL=$(python -c "import nvidia.nccl;print(list(nvidia.nccl.__path__)[0])")
mkdir -p build/dbg
for f in ccl_kernels ccl_api ccl_sharded; do
  nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -Xcompiler -fPIC -DCCL_DEBUG_PRINT \
    -I include -I paper_1606_05973_b200/csrc -I $NCCL/include -c paper_1606_05973_b200/csrc/$f.cu -o build/dbg/$f.o
done
nvcc -gencode arch=compute_100a,code=sm_100a -shared -o paper_1606_05973_b200/libccl_b200_dbg.so build/dbg/*.o -L $NCCL/lib -l:libnccl.so.2 -Xlinker -rpath=$NCCL/lib -lcudart
