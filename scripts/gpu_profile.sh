#!/bin/bash
# Round profiling run on one B200 (see /opt/skills/guides/B200_PROFILING.md):
#   1. the default bench line (config 5) and bench lines of configs 1-4, the int64 config-5 line and
#      the single-image latency table, 2. the ncu launch list of the default command,
#   3. full ncu captures of the dominant kernels (tail, largest write pass) on config 5, with the
#      library's per-launch algorithmic bytes of the same run (run_once.py prints them).
set -x
mkdir -p gpurun_out
sha256sum paper_1007_0547_b200/libhht.so > gpurun_out/libhht.sha256
python -c "from paper_1007_0547_b200 import hht; print(hht.version())" > gpurun_out/libhht.version
python bench.py > gpurun_out/bench_default.log 2> gpurun_out/bench_default.err && \
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
    --log-file gpurun_out/launches_c5.csv python bench.py > gpurun_out/ncu_launches.log 2>&1
echo "launch list rc=$?"
for c in 1 2; do python bench.py --config $c --steps 200 --warmup 20 > gpurun_out/bench_c$c.log 2> gpurun_out/bench_c$c.err; done
python bench.py --config 3 --steps 20 --warmup 5 > gpurun_out/bench_c3.log 2> gpurun_out/bench_c3.err
python bench.py --config 4 --steps 5 --warmup 3 > gpurun_out/bench_c4.log 2> gpurun_out/bench_c4.err
python bench.py --force-int64 --no-cpu-baseline > gpurun_out/bench_c5_int64.log 2> gpurun_out/bench_c5_int64.err
python scripts/latency_bench.py --out gpurun_out/latency.md > gpurun_out/latency.log 2>&1
python scripts/run_once.py --config 5 > gpurun_out/plain_c5.log 2>&1
# k_pass launch index of the largest write pass (k_pass launch 0 is the root count pass)
WSKIP=$(python -c "
import ast,re
t=open('gpurun_out/plain_c5.log').read()
b=ast.literal_eval(re.search(r'^write launches \d+ first bytes \d+ bytes\[:16\] (\[.*\])$', t, re.M).group(1))
print(1 + max(range(len(b)), key=lambda i: b[i]))")
echo "write capture index $WSKIP" > gpurun_out/write_skip.txt
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_tail|k_fused" -c 1 \
    -o gpurun_out/c5_tail python scripts/run_once.py --config 5 > gpurun_out/ncu_tail.log 2>&1
echo "tail capture rc=$?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_pass -s $WSKIP -c 1 \
    -o gpurun_out/c5_write python scripts/run_once.py --config 5 > gpurun_out/ncu_write.log 2>&1
echo "write capture rc=$?"
# the largest count-ahead list pass (MODE_WRITE: write launch 6 of config 5, level 6 -> lists of 7, votes of 8)
timeout 900 ncu --set full --clock-control none --import-source on --kernel-name-base demangled \
    -k regex:"k_pass<int, \\(int\\)1," -s 6 -c 1 \
    -o gpurun_out/c5_write_ca python scripts/run_once.py --config 5 > gpurun_out/ncu_write_ca.log 2>&1
echo "count-ahead capture rc=$?"
# edge front end (NEXT-3) on the same build
python scripts/frontend_bench.py --out gpurun_out/frontend.md > gpurun_out/frontend.log 2>&1
echo "frontend rc=$?"
# counters of this build into profiles/ncu_traffic.json (on the box), then the default bench line
# again so that roofline.traffic carries them (bench.py attaches counters only by build id)
python scripts/ncu_summary.py --round 2 > gpurun_out/ncu_summary.log 2>&1 && \
python bench.py > gpurun_out/bench_default.log 2> gpurun_out/bench_default.err
echo "bench with traffic rc=$?"
