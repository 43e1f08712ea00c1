#!/bin/bash
# Interleaved A/B of library builds on the config-2 headline (bench.py, 1000-step
# graph replays):  tools/ab_libs.sh REPS TAG1 TAG2 ...  (TAG = libntt_b200_TAG.so; "cur" = the default)
REPS=$1; shift
for i in $(seq $REPS); do
  for t in "$@"; do
    if [ "$t" = cur ]; then L=; else L=paper_2405_11353_b200/libntt_b200_$t.so; fi
    echo "$t $(NTT_LIB_PATH=$L python bench.py --steps 1000 --warmup 10 --no-cpu --no-extra 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print(round(d['ms_per_step']*1e3,2), round(d['roofline']['frac'],3), 'dit', round(d['dit']['roofline_frac'],3), d['sha256_parity'], d['dit']['sha256_parity'])")"
  done
done
