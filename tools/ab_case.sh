#!/bin/bash
# Interleaved A/B of one workload across library builds (tools/build_variant.sh):
#   tools/ab_case.sh REPS CFG "VARIANTS" TAG...   ("cur" = the default library)
REPS=$1; CFG=$2; VARS=$3; shift 3
for i in $(seq $REPS); do
  for t in "$@"; do
    if [ "$t" = cur ]; then L=; else L=paper_2405_11353_b200/libntt_b200_$t.so; fi
    for v in $VARS; do echo "$t $(NTT_LIB_PATH=$L python tools/time_case.py $CFG $v 20 2>&1 | tail -1)"; done
  done
done
