#!/bin/bash
# build librk variants for tools/variant_bench.py: name:flags ...
cd "$(dirname "$0")/.."
for spec in "$@"; do
  name=${spec%%:*}; flags=${spec#*:}
  /usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -shared -Xcompiler -fPIC \
    -I include -I paper_1511_07983_b200/csrc $flags -o build_var/librk_$name.so \
    paper_1511_07983_b200/csrc/rk_host.cpp paper_1511_07983_b200/csrc/rk_kernels.cu -Xptxas -v 2>&1 | \
    grep -A2 "rk_eval_kernelILi${VARIANT:-2}ELb1" | grep -E "Used|spill" | sed "s/^/$name: /"
done
