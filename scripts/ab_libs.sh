#!/bin/bash
# A/B of libhht.so build variants on one GPU: for each paper_1007_0547_b200/libhht_<tag>.so given,
# install it as libhht.so and run the default bench line (device time only).
mkdir -p gpurun_out
for tag in "$@"; do
  cp paper_1007_0547_b200/libhht_$tag.so paper_1007_0547_b200/libhht.so
  timeout 300 python bench.py --no-cpu-baseline --no-e2e > gpurun_out/ab_$tag.log 2> gpurun_out/ab_$tag.err
  echo "$tag rc=$?"
done
