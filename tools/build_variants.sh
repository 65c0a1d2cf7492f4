#!/bin/bash
# Build experiment variants of the library next to the product one.
set -e
cd "$(dirname "$0")/.."
P=paper_2503_12204_b200
python $P/build.py -DD4K_PHILOX_ROUNDS=7 --out=$P/libd4orm_exp_r7.so &
python $P/build.py -DD4K_EXPERIMENT_CHEAP_RNG --out=$P/libd4orm_exp_cheap.so &
python $P/build.py -DD4K_EXPERIMENT_SKIP_B --out=$P/libd4orm_exp_skipb.so &
wait
