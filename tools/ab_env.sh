#!/bin/bash
# Interleaved A/B of an environment switch on the config-2 headline (bench.py graph replays):
#   tools/ab_env.sh REPS VAR VAL1 VAL2 ...
REPS=$1; VAR=$2; shift 2
for i in $(seq $REPS); do
  for v in "$@"; do
    echo "$VAR=$v $(env $VAR=$v python bench.py --steps 1000 --warmup 10 --no-cpu --no-extra --no-sweep 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print(round(d['ms_per_step']*1e3,2), round(d['roofline']['frac'],3), 'dit', round(d['dit']['roofline_frac'],3), d['sha256_parity'], d['dit']['sha256_parity'])")"
  done
done
