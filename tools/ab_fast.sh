# A/B of fast-kernel build variants on config 2 (1000-step graph replays):
#   tools/build_variant.sh TAG k_f32s.cu -D...;  bash tools/ab_fast.sh TAG...
for i in ${REPS:-1 2 3}; do for T in base "$@"; do
  L=; [ "$T" != base ] && L=paper_2405_11353_b200/libntt_b200_$T.so
  echo "$T $(NTT_LIB_PATH=$L python bench.py --steps 1000 --warmup 10 --no-cpu --no-extra --no-sweep 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print(round(d['ms_per_step']*1e3,2), round(d['roofline']['frac'],3), round(d['dit']['roofline_frac'],3), d['sha256_parity'], d['dit']['sha256_parity'])")"
done; done
