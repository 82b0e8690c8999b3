#!/bin/bash
# Builds a variant of libed_gpu.so with extra -D flags for one source
# (development experiments): tools/build_variant.sh NAME SRC.cu -DFOO=1 ...
# -> paper_2410_02682_b200/build/var/NAME.so (load with ED_LIB_PATH=...).
set -e
cd "$(dirname "$0")/.."
NAME=$1; SRC=$2; shift 2
P=paper_2410_02682_b200
python -c "from paper_2410_02682_b200 import build as b; b.build()"
mkdir -p $P/build/var
OBJS=""
for s in runtime gemm_sm100 kernels ewise attn_sm100; do
  if [ "$s.cu" = "$SRC" ]; then
    /usr/local/cuda/bin/nvcc -std=c++17 -O3 -lineinfo -Xcompiler -fPIC -Xcompiler -fvisibility=hidden -Iinclude -I$P/csrc \
      -gencode arch=compute_100a,code=sm_100a "$@" -c $P/csrc/$s.cu -o $P/build/var/$NAME.$s.o
    OBJS="$OBJS $P/build/var/$NAME.$s.o"
  else
    OBJS="$OBJS $P/build/$s.o"
  fi
done
/usr/local/cuda/bin/nvcc -shared -gencode arch=compute_100a,code=sm_100a $OBJS -o $P/build/var/$NAME.so -lcudart -lnccl \
  -Xlinker /usr/lib/x86_64-linux-gnu/libstdc++.so.6
echo $P/build/var/$NAME.so
