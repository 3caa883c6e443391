#!/bin/bash
# Round-2 ncu evidence (run under gpurun). Every capture is summarised ON THE BOX into gpurun_out/profiles_r2/
# (raw metric CSV, SASS summary, per-source-line profile) and the .ncu-rep is dropped: six reports with imported
# sources exceed what gpurun copies back.
set -x
OUT=gpurun_out/profiles_r2
mkdir -p $OUT /tmp/prof
NCU="ncu --set full --clock-control none --import-source on"
LIB=paper_2603_15780_b200/lib/libdigeo_b200.so
(cd /tmp/prof && cuobjdump -xelf dg_trace_kernel.sm_100a.cubin $OLDPWD/$LIB > /dev/null && nvdisasm -g -c dg_trace_kernel.sm_100a.cubin > /tmp/prof/trace_dis.txt)
capture() {  # name, launches of trace_fast_kernel to skip, mangled-name substring for the line profile, command...
  local name=$1 skip=$2 mangled=$3; shift 3
  if [ -n "$ONLY" ] && [[ ! " $ONLY " =~ " $name " ]]; then return; fi
  $NCU -k regex:trace_fast_kernel -s $skip -c 1 -f -o /tmp/prof/$name "$@" > $OUT/$name.log 2>&1
  ncu -i /tmp/prof/$name.ncu-rep --page raw --csv > $OUT/${name}_raw.csv 2>/dev/null
  ncu -i /tmp/prof/$name.ncu-rep --page source --csv --print-source sass > /tmp/prof/${name}_sass.csv 2>/dev/null
  python profiles/ncu_sass_summary.py /tmp/prof/${name}_sass.csv > $OUT/${name}_sass_summary.txt 2>&1
  python profiles/ncu_line_profile.py /tmp/prof/${name}_sass.csv /tmp/prof/trace_dis.txt "$mangled" > $OUT/${name}_line_profile.txt 2>&1
  rm -f /tmp/prof/$name.ncu-rep /tmp/prof/${name}_sass.csv
}
capture r2_c2_forward          2 "trace_fast_kernelILb1ELi0ELi0ELb0ELi0ELb0E" python scripts/profile_target.py c2 forward exact
capture r2_c2_forward_fastlane 2 "trace_fast_kernelILb1ELi0ELi0ELb0ELi1ELb0E" python scripts/profile_target.py c2 forward fast
capture r2_c3_forward          2 "trace_fast_kernelILb1ELi0ELi0ELb0ELi0ELb0E" python scripts/profile_target.py c3 forward exact
# (a fused call launches the walker three times: seeds, round 2, par jobs -- the eighth launch is round 2 of call 3)
capture r2_c3_fused_gfd        7 "trace_fast_kernelILb1ELi0ELi0ELb1ELi0ELb0E" python scripts/profile_target.py c3 fused exact
capture r2_c4_forward          2 "trace_fast_kernelILb1ELi0ELi0ELb0ELi0ELb0E" python scripts/profile_target.py c4 forward exact
# (a batch in start-face order on a mesh beyond 250 MB of records is queued on both gathers, one of which returns at
# once: c3 / c4 run the per-lane loads -- the third launch is call 2's --, config 5's long traces the cooperative
# gather: the sixth launch is call 3's)
capture r2_c5_forward          5 "trace_fast_kernelILb1ELi2ELi0ELb0ELi0ELb0E" python scripts/profile_target.py c5 forward exact
if [ -n "$ONLY" ]; then ls -la $OUT; exit 0; fi
# every launch of a short default bench run with its device time (cold-cache, serialised: compare SHARES)
ncu --metrics gpu__time_duration.sum --clock-control none -c 600 --csv --log-file $OUT/r2_launches_bench.csv \
    python bench.py --steps 2 --warmup 3 --no-cpu > $OUT/r2_launches_bench.log 2>&1
ls -la $OUT
