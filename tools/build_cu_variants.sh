#!/bin/bash
# Variants of the library that differ only in d4orm_cuda.cu's object:
# tools/build_cu_variants.sh NAME "-DFLAG ..." [NAME "-D..."]...  ->  paper_2503_12204_b200/libd4orm_exp_NAME.so
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
  nvcc -gencode arch=compute_100a,code=sm_100a $INC $DEFS -c $P/csrc/d4orm_cuda.cu -o /tmp/d4orm_cuda_$NAME.o &
  PIDS="$PIDS $!"; NAMES="$NAMES $NAME"
done
wait
for NAME in $NAMES; do
  OBJS=$(ls $P/build/*.o | grep -v d4orm_cuda.cu.o)
  nvcc -gencode arch=compute_100a,code=sm_100a -shared -o $P/libd4orm_exp_$NAME.so $OBJS /tmp/d4orm_cuda_$NAME.o -ldl -lcudart
  echo built $P/libd4orm_exp_$NAME.so
done
