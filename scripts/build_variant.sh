#!/bin/bash
# Build paper_1007_0547_b200/libhht_<tag>.so with extra nvcc flags (A/B experiments, scripts/ab_libs.sh).
#   bash scripts/build_variant.sh <tag> [-DNAME=VALUE ...]
set -e
tag=$1; shift
ND=$(python -c "import nvidia.nccl,os; print(list(nvidia.nccl.__path__)[0])")
C=paper_1007_0547_b200/csrc
/usr/local/cuda/bin/nvcc -std=c++17 -O3 -lineinfo -shared -Xcompiler -fPIC -gencode arch=compute_100a,code=sm_100a \
  -I include -I $C -I $ND/include "$@" -o paper_1007_0547_b200/libhht_$tag.so \
  $C/hht_kernels.cu $C/hht_mid.cu $C/hht_driver.cu -L $ND/lib -l:libnccl.so.2 -Xlinker=-rpath=$ND/lib
echo built paper_1007_0547_b200/libhht_$tag.so
