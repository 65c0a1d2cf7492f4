#!/bin/bash
# Build K2+K3 variants of the library that differ only in the k23_k*.cu objects:
# tools/build_pl32_variants.sh NAME "-DFLAG ..." [NAME "-D..."]...  ->  paper_2503_12204_b200/libd4orm_exp_NAME.so
set -e
cd "$(dirname "$0")/.."
P=paper_2503_12204_b200
INC=$(python - <<'PY'
import sys
sys.path.insert(0, '.')
from paper_2503_12204_b200 import build as b
print(" ".join(b.NVCC_FLAGS))
PY
)
while [ $# -ge 2 ]; do
  NAME=$1; DEFS=$2; shift 2
  D=$P/build_exp_$NAME; mkdir -p $D
  for k in 0 1 2 3 4 5; do
    nvcc -gencode arch=compute_100a,code=sm_100a $INC $DEFS -c $P/csrc/k23_k$k.cu -o $D/k23_k$k.cu.o &
  done
  wait
  OBJS=$(ls $P/build/*.o | grep -v k23_k)
  nvcc -gencode arch=compute_100a,code=sm_100a -shared -o $P/libd4orm_exp_$NAME.so $OBJS $D/k23_k*.cu.o -ldl -lcudart
  rm -rf $D
  echo built $P/libd4orm_exp_$NAME.so
done
