#!/bin/bash
# A/B of libhht.so build variants on the end-to-end path (scripts/e2e_breakdown.py per variant).
#   bash scripts/ab_e2e.sh <tag> ...   (each paper_1007_0547_b200/libhht_<tag>.so)
mkdir -p gpurun_out
for tag in "$@"; do
  cp paper_1007_0547_b200/libhht_$tag.so paper_1007_0547_b200/libhht.so
  timeout 600 python scripts/e2e_breakdown.py --reps 5 > gpurun_out/e2e_$tag.log 2>&1
  echo "== $tag"; grep -E "packed|cap 0|no sink" gpurun_out/e2e_$tag.log
done
