#!/bin/bash
# build_variant.sh NAME "NVCC -D flags" [files]: librbf with the given csrc files (default
# summation.cu) recompiled under the flags, at paper_1305_5179_b200/variants/librbf_NAME.so
# (tuning experiments; tools/bench_kernels.py --lib, tools/sessions/sess_var.sh)
set -e
cd "$(dirname "$0")/.."
python -m paper_1305_5179_b200.build >/dev/null
cd paper_1305_5179_b200
mkdir -p variants
files=${3:-summation.cu}
objs=""
for f in $(ls build/*.o); do
  b=$(basename $f .o)
  if [[ " $files " == *" $b.cu "* ]]; then
    nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++20 -Xcompiler -fPIC,-ffp-contract=off -diag-suppress 177 $2 -c -o variants/${b}_$1.o csrc/$b.cu
    objs="$objs variants/${b}_$1.o"
  else
    objs="$objs $f"
  fi
done
nvcc -gencode arch=compute_100a,code=sm_100a -shared -o variants/librbf_$1.so $objs
echo variants/librbf_$1.so
