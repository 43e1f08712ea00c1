for t in "$@"; do if [ $t = base ]; then L=; else L=paper_2405_11353_b200/libntt_b200_$t.so; fi; echo "$t $(NTT_LIB_PATH=$L python tools/time_case.py 4 pease_nc 20)"; done
