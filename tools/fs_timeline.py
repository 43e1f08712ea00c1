"""Where a four-step pass CTA spends its clocks (library built with -DNTT_FS_TIMELINE:
tools/build_variant.sh fstl kfs_f32.cu -DNTT_FS_TIMELINE):
    NTT_LIB_PATH=paper_2405_11353_b200/libntt_b200_fstl.so python tools/fs_timeline.py [CFG] [VARIANT]
Thread 0 of every CTA sums clock64() deltas between phase boundaries over all its tiles."""
import ctypes, os, sys
import numpy as np, torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2405_11353_b200 as P
from paper_2405_11353_b200 import _lib
from paper_2405_11353_b200.configs import CONFIGS, seeded_input
cfg = int(sys.argv[1]) if len(sys.argv) > 1 else 4
variant = sys.argv[2] if len(sys.argv) > 2 else "pease_nc"
w = CONFIGS[cfg]
plan = P.make_plan(P.FieldParams(w.p, w.g, w.w), variant, w.n, n1=w.n1)
dp = P.algorithms.device_plan_for(plan, w.word, 0)
x = torch.from_numpy(seeded_input(w).view(np.int32)).view(torch.uint32).cuda()
y = torch.empty_like(x)
s = torch.cuda.current_stream().cuda_stream
for _ in range(3): dp.exec_device(x.data_ptr(), y.data_ptr(), w.batch, False, s)
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record(); dp.exec_device(x.data_ptr(), y.data_ptr(), w.batch, False, s); e1.record(); torch.cuda.synchronize()
print(f"cfg{cfg} {variant}: {e0.elapsed_time(e1)*1e3:.1f} us (instrumented build)")
L = _lib.load()
n = 2 * 1024 * 8
buf = (ctypes.c_ulonglong * n)()
L.ntt_debug_fs_timeline.argtypes = [ctypes.c_void_p, ctypes.c_int]
assert L.ntt_debug_fs_timeline(buf, n) == 0
a = np.array(buf, dtype=np.uint64).reshape(2, 1024, 8).astype(np.float64)
names = ["store drain / loop top", "wait for the tile (mbarrier)", "group 0 (reads, butterflies, barrier, writes)",
         "twist factors + next-tile issue + barrier", "middle groups", "last group reads + butterflies", "twist + stores"]
for mode in (0, 1):
    m = a[mode]; m = m[m[:, 7] > 0]
    if not len(m): continue
    tiles = m[:, 7]
    tot = m[:, :7].sum(axis=1)
    print(f"pass {'AB'[mode]}: {len(m)} CTAs, {tiles.mean():.1f} tiles each, {np.median(tot / tiles):.0f} clocks per tile per CTA")
    for k, nm in enumerate(names):
        per = m[:, k] / tiles
        print(f"  {nm:48s} p50 {np.median(per):7.0f} clk  {100 * m[:, k].sum() / tot.sum():5.1f} %")
