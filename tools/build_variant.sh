#!/bin/bash
# Builds a variant of libed_gpu.so for A/B experiments: one translation unit
# compiled from SRC (a path, e.g. an older revision saved under /tmp, or the
# tree's own file) with extra -D flags, every other object from the current
# build: tools/build_variant.sh NAME UNIT SRC.cu -DFOO=1 ...
# -> paper_2410_02682_b200/build/var/NAME.so (load with ED_LIB_PATH=...).
set -e
cd "$(dirname "$0")/.."
NAME=$1; UNIT=$2; SRC=$3; shift 3
P=paper_2410_02682_b200
python -c "from paper_2410_02682_b200 import build as b; b.build()"
mkdir -p $P/build/var
OBJS=""
for s in $(python -c "from paper_2410_02682_b200 import build as b; print(' '.join(x[:-3] for x in b.SOURCES))"); do
  if [ "$s" = "$UNIT" ]; then
    /usr/local/cuda/bin/nvcc -std=c++17 -O3 -lineinfo -Xcompiler -fPIC -Xcompiler -fvisibility=hidden -Iinclude \
      -I$(dirname $SRC) -I$P/csrc -gencode arch=compute_100a,code=sm_100a "$@" -c $SRC -o $P/build/var/$NAME.$s.o
    OBJS="$OBJS $P/build/var/$NAME.$s.o"
  else
    OBJS="$OBJS $P/build/$s.o"
  fi
done
/usr/local/cuda/bin/nvcc -shared -gencode arch=compute_100a,code=sm_100a $OBJS -o $P/build/var/$NAME.so -lcudart -lnccl \
  -Xlinker /usr/lib/x86_64-linux-gnu/libstdc++.so.6
echo $P/build/var/$NAME.so
