set -x
OUT=gpurun_out/profiles_r2; mkdir -p $OUT /tmp/prof
LIB=paper_2603_15780_b200/lib/libdigeo_b200.so
(cd /tmp/prof && cuobjdump -xelf dg_trace_kernel.sm_100a.cubin $OLDPWD/$LIB > /dev/null && nvdisasm -g -c dg_trace_kernel.sm_100a.cubin > /tmp/prof/trace_dis.txt)
name=r2_c5_vertex_generic
python scripts/dev/c5_vertex_generic.py 100000 > $OUT/$name.plain.log 2>&1 || exit 1
ncu --set full --clock-control none --import-source on -k regex:trace_kernel -s 2 -c 1 -f -o /tmp/prof/$name python scripts/dev/c5_vertex_generic.py 100000 > $OUT/$name.log 2>&1
ncu -i /tmp/prof/$name.ncu-rep --page raw --csv > $OUT/${name}_raw.csv 2>/dev/null
ncu -i /tmp/prof/$name.ncu-rep --page source --csv --print-source sass > /tmp/prof/${name}_sass.csv 2>/dev/null
python profiles/ncu_sass_summary.py /tmp/prof/${name}_sass.csv > $OUT/${name}_sass_summary.txt 2>&1
python profiles/ncu_line_profile.py /tmp/prof/${name}_sass.csv /tmp/prof/trace_dis.txt "trace_kernelIdLb0ELb1E" > $OUT/${name}_line_profile.txt 2>&1
head -40 $OUT/${name}_sass_summary.txt
