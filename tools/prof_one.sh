#!/bin/bash
# usage (on the GPU box): bash tools/prof_one.sh NAME CFG VARIANT KERNEL_REGEX COUNT [inv]
set -u
OUT=gpurun_out/p1; mkdir -p $OUT
python tools/prof_case.py $2 $3 3 ${6:-} > $OUT/$1_plain.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:$4 -s $5 -c $5 -o $OUT/$1 \
    python tools/prof_case.py $2 $3 3 ${6:-} > $OUT/$1_ncu.log 2>&1
ncu -i $OUT/$1.ncu-rep --page raw --csv > $OUT/$1_raw.csv 2>/dev/null
ncu -i $OUT/$1.ncu-rep --page source --csv --print-source sass > $OUT/$1_sass.csv 2>/dev/null
gzip -f $OUT/$1_sass.csv; rm -f $OUT/$1.ncu-rep
