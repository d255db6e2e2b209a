#!/bin/bash
# Timing-only A/B of libhht.so build variants (no parity: for experiments that change results).
mkdir -p gpurun_out
for tag in "$@"; do
  cp paper_1007_0547_b200/libhht_$tag.so paper_1007_0547_b200/libhht.so
  timeout 300 python bench.py --no-cpu-baseline --no-e2e > gpurun_out/ab_$tag.log 2> gpurun_out/ab_$tag.err
  python -c "
import json; l=[x for x in open('gpurun_out/ab_$tag.log') if x.startswith('{')][-1]; j=json.loads(l); print('$tag', round(j['ms_per_step'],2), 'tail', round(j['kernel_ms']['tail'],2), 'write', round(j['kernel_ms']['write'],2))" 2>&1 | tail -1
done
