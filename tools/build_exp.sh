#!/bin/bash
# Build experiment variants of the library (tools/_exp/<name>.so) with extra
# -D flags, e.g.  tools/build_exp.sh noconv -DRGB_EXP_NOCONV
set -e
cd "$(dirname "$0")/../paper_1503_02852_b200"
name=$1; shift
mkdir -p ../tools/_exp
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -Xcompiler -fPIC -shared "$@" \
  -o ../tools/_exp/$name.so csrc/rgb_kernels.cu csrc/rgb_tc_gemm.cu csrc/rgb_scc.cu csrc/rgb_plan.cu csrc/rgb_prof.cu csrc/rgb_comm.cu -ldl
