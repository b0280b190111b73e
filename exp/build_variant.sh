#!/bin/bash
# build_variant.sh NAME SRC.cu [FILE.cu] : libslora_b200 with FILE.cu (default attn_prefill.cu)
# replaced by SRC.cu -> exp/NAME.so
set -e
cd /root/repo/paper_2505_14468_b200/csrc
FILE=${3:-attn_prefill.cu}
BASE=${FILE%.cu}
NV="nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -Xcompiler -fPIC -Xcompiler -fvisibility=hidden -I/opt/prime-rl/.venv/lib/python3.12/site-packages/nvidia/nccl/include --expt-relaxed-constexpr"
cp "$2" ./_variant.cu
$NV -c _variant.cu -o build/_variant.o
rm -f _variant.cu
OBJS=$(ls build/*.o | grep -v "/$BASE.o" | grep -v _variant)
nvcc -gencode arch=compute_100a,code=sm_100a $OBJS build/_variant.o -shared -L/opt/prime-rl/.venv/lib/python3.12/site-packages/nvidia/nccl/lib -l:libnccl.so.2 -Xlinker -rpath=/opt/prime-rl/.venv/lib/python3.12/site-packages/nvidia/nccl/lib -cudart static -o /root/repo/exp/$1.so
rm -f build/_variant.o
