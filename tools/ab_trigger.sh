# A/B of the fast kernel trigger order: build the variant first with
#   tools/build_variant.sh tf k_f32s.cu -DNTT_FAST_TRIGGER_FIRST=0
for i in 1 2 3 4 5; do for L in "" paper_2405_11353_b200/libntt_b200_tf.so; do echo "lib=$L $(NTT_LIB_PATH=$L python bench.py --steps 1000 --warmup 10 --no-cpu --no-extra --no-sweep 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print(round(d[\"ms_per_step\"]*1e3,2), round(d[\"roofline\"][\"frac\"],3), round(d[\"dit\"][\"roofline_frac\"],3))")"; done; done
