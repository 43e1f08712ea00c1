#!/bin/bash
# Run ON the GPU box (gpurun): ncu launch list of the bench command + one
# `--set full` capture per workload's top kernel.  Each ncu command runs only
# after the same command exited 0 without ncu.
set -u
OUT=gpurun_out/prof
mkdir -p $OUT
BENCH="python bench.py --steps 5 --warmup 3 --no-cpu --no-extra"
$BENCH > $OUT/bench_plain.log 2>&1 && \
  ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $OUT/launches.csv $BENCH > $OUT/bench_ncu.log 2>&1
cap() {  # name kernel-regex cfg variant [inv]
  python tools/prof_case.py $3 $4 3 ${5:-} > $OUT/$1_plain.log 2>&1 && \
    ncu --set full --clock-control none --import-source on -k regex:$2 -s 2 -c ${6:-1} -o $OUT/$1 \
      python tools/prof_case.py $3 $4 3 ${5:-} > $OUT/$1_ncu.log 2>&1
  if [ -f $OUT/$1.ncu-rep ]; then
    ncu -i $OUT/$1.ncu-rep --page raw --csv > $OUT/$1_raw.csv 2>/dev/null
    ncu -i $OUT/$1.ncu-rep --page source --csv --print-source sass > $OUT/$1_sass.csv 2>/dev/null
    gzip -f $OUT/$1_sass.csv
    sz=$(stat -c %s $OUT/$1.ncu-rep)
    if [ "$sz" -gt 8000000 ]; then rm -f $OUT/$1.ncu-rep; echo "$1: rep $sz bytes dropped" >> $OUT/dropped.txt; fi
  fi
}
cap c2_pease_nc k_fast 2 pease_nc
cap c2_dit k_fast 2 dit
cap c3_dif k_fs 3 dif "" 2
cap c4_pease_nc "k_fs" 4 pease_nc "" 2
cap c5_sixstep "k_cols|k_tile" 5 sixstep "" 4
echo profile_round done
