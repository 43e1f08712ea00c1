#!/bin/bash
# Run ON the GPU box (gpurun): one `--set full` capture per workload's top
# kernels (after the same command exited 0 without ncu); raw + SASS source pages.
set -u
OUT=gpurun_out/prof_r2
mkdir -p $OUT
cap() {  # name kernel-regex cfg variant [inv] [count]
  python tools/prof_case.py $3 $4 3 ${5:-} > $OUT/$1_plain.log 2>&1 && \
    ncu --set full --clock-control none --import-source on -k regex:$2 -s ${7:-2} -c ${6:-1} -o $OUT/$1 \
      python tools/prof_case.py $3 $4 3 ${5:-} > $OUT/$1_ncu.log 2>&1
  if [ -f $OUT/$1.ncu-rep ]; then
    ncu -i $OUT/$1.ncu-rep --page raw --csv > $OUT/$1_raw.csv 2>/dev/null
    ncu -i $OUT/$1.ncu-rep --page source --csv --print-source sass > $OUT/$1_sass.csv 2>/dev/null
    gzip -f $OUT/$1_sass.csv
    sz=$(stat -c %s $OUT/$1.ncu-rep)
    if [ "$sz" -gt 8000000 ]; then rm -f $OUT/$1.ncu-rep; echo "$1: rep $sz bytes dropped" >> $OUT/dropped.txt; fi
  fi
}
for c in "$@"; do
  case $c in
    c2) cap c2_pease_nc k_fast 2 pease_nc ;;
    c3) cap c3_dif k_fs 3 dif "" 2 ;;
    c4) cap c4_pease_nc k_fs 4 pease_nc "" 2 ;;
    c5) cap c5_sixstep "k_cols|k_tile|k_transpose" 5 sixstep "" 5 5 ;;
  esac
done
echo prof_r2 done
