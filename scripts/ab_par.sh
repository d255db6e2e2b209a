#!/bin/bash
# A/B of libhht.so build variants: a parity subset (fused tail, work units, full configs) and the
# default bench line (device time only) per variant.   bash scripts/ab_par.sh <tag> ...
mkdir -p gpurun_out
for tag in "$@"; do
  cp paper_1007_0547_b200/libhht_$tag.so paper_1007_0547_b200/libhht.so
  timeout 600 python -m pytest tests/test_gpu_parity.py -q -x -k "tail_depth or work_units or raster_fixed or config_full" > gpurun_out/ab_par_$tag.log 2>&1
  echo "$tag parity rc=$? $(tail -1 gpurun_out/ab_par_$tag.log)"
  timeout 300 python bench.py --no-cpu-baseline --no-e2e > gpurun_out/ab_$tag.log 2> gpurun_out/ab_$tag.err
  python -c "
import json; l=[x for x in open('gpurun_out/ab_$tag.log') if x.startswith('{')][-1]; j=json.loads(l); print('$tag', round(j['ms_per_step'],2), 'tail', round(j['kernel_ms']['tail'],2), 'write', round(j['kernel_ms']['write'],2))"
done
