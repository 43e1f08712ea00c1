#!/bin/bash
# Run ON the GPU box: steady-state DRAM traffic and time per step of every bench workload
# (ncu app-range replay over 16 back-to-back steps, tools/traffic_range.py), after the same
# command exited 0 without ncu.  tools/traffic_summary.py turns the CSVs into profiles/<round>/traffic_steady.json.
OUT=gpurun_out/traffic; mkdir -p $OUT
run() {  # name cfg variant
  python tools/traffic_range.py $2 $3 16 > $OUT/$1_plain.log 2>&1 && \
  ncu --replay-mode app-range --clock-control none --csv --log-file $OUT/$1.csv \
      --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum,lts__t_sectors_srcunit_tex_op_read_lookup_hit.sum,lts__t_sectors_srcunit_tex_op_read.sum \
      python tools/traffic_range.py $2 $3 16 > $OUT/$1_ncu.log 2>&1
}
run config2_pease_nc 2 pease_nc
run config2_dit 2 dit
run config3_dif 3 dif
run config4_pease_nc 4 pease_nc
run config5_sixstep 5 sixstep
echo traffic_all done
