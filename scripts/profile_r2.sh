#!/bin/bash
# Round-2 ncu evidence (run under gpurun; reports land in gpurun_out/, summaries are made from them into profiles/).
set -x
NCU="ncu --set full --clock-control none --import-source on"
$NCU -k regex:trace_fast_kernel -s 2 -c 1 -o gpurun_out/r2_c2_forward            python scripts/profile_target.py c2 forward exact
$NCU -k regex:trace_fast_kernel -s 2 -c 1 -o gpurun_out/r2_c2_forward_fastlane   python scripts/profile_target.py c2 forward fast
$NCU -k regex:trace_fast_kernel -s 2 -c 1 -o gpurun_out/r2_c3_forward            python scripts/profile_target.py c3 forward exact
$NCU -k "regex:trace_fast_kernel<1, 0, 0, 1" -s 2 -c 1 -o gpurun_out/r2_c3_fused_gfd  python scripts/profile_target.py c3 fused exact
$NCU -k regex:trace_fast_kernel -s 2 -c 1 -o gpurun_out/r2_c4_forward            python scripts/profile_target.py c4 forward exact
$NCU -k regex:trace_fast_kernel -s 2 -c 1 -o gpurun_out/r2_c5_forward            python scripts/profile_target.py c5 forward exact 500000
# every launch of a short default bench run with its device time (cold-cache, serialised: compare SHARES)
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/r2_launches_bench.csv \
    python bench.py --steps 2 --warmup 3 --no-cpu > gpurun_out/r2_launches_bench.log 2>&1
