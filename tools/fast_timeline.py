"""Per-CTA phase timeline of the single-pass kernel (library built with
-DNTT_FAST_TIMELINE: tools/build_variant.sh tl k_f32s.cu -DNTT_FAST_TIMELINE):
    NTT_LIB_PATH=paper_2405_11353_b200/libntt_b200_tl.so python tools/fast_timeline.py [CFG] [VARIANT]
Slots per (CTA, team): 0 entry, 1 table copied, 2 after griddepcontrol.wait, 3 first
polynomial landed, 4 first polynomial stored, 5 exit, 7 the previous launch's exit."""
import ctypes, os, sys
import numpy as np, torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2405_11353_b200 as P
from paper_2405_11353_b200 import _lib
from paper_2405_11353_b200.configs import CONFIGS, seeded_input
cfg = int(sys.argv[1]) if len(sys.argv) > 1 else 2
variant = sys.argv[2] if len(sys.argv) > 2 else "pease_nc"
w = CONFIGS[cfg]
plan = P.make_plan(P.FieldParams(w.p, w.g, w.w), variant, w.n, n1=w.n1)
dp = P.algorithms.device_plan_for(plan, w.word, 0)
x0 = torch.from_numpy(seeded_input(w).view(np.int32)).view(torch.uint32).cuda()
xs = [x0.clone() for _ in range(4)]
ys = [torch.empty_like(x0) for _ in range(4)]
st = torch.cuda.Stream()
K = 12
with torch.cuda.stream(st):
    for i in range(4): dp.exec_device(xs[i % 4].data_ptr(), ys[i % 4].data_ptr(), w.batch, False, st.cuda_stream, independent=True)
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g, stream=st):
        for i in range(K): dp.exec_device(xs[i % 4].data_ptr(), ys[i % 4].data_ptr(), w.batch, False, st.cuda_stream, independent=True)
    g.replay(); torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(st); g.replay(); e1.record(st); torch.cuda.synchronize()
print(f"graph: {e0.elapsed_time(e1) / K * 1e3:.2f} us/step")
L = _lib.load()
buf = (ctypes.c_ulonglong * (256 * 64))()
L.ntt_debug_timeline.argtypes = [ctypes.c_void_p, ctypes.c_int]
assert L.ntt_debug_timeline(buf, 256 * 64) == 0
a = np.array(buf, dtype=np.uint64).reshape(256, 8, 8).astype(np.int64)
a = a[a[:, 0, 0] > 0]
print(len(a), 'SMs')
teams = 4 if cfg == 2 else int((a[0, :, 0] > 0).sum())
a = a[:, :teams, :]
t0 = a[:, :, 0].min()
rel = lambda k: (a[:, :, k] - t0) / 1e3
def show(name, v):
    print(f"{name:44s} min {v.min():7.2f}  p50 {np.median(v):7.2f}  max {v.max():7.2f} us")
show("entry after the first CTA's entry", rel(0))
show("same SM: previous exit -> this entry", (a[:, :, 0] - a[:, :, 7]) / 1e3)
show("last exit of the previous launch -> entry", (a[:, :, 0] - a[:, :, 7].max()) / 1e3)
show("table copy + barrier init (0 -> 1)", (a[:, :, 1] - a[:, :, 0]) / 1e3)
show("griddepcontrol.wait (1 -> 2)", (a[:, :, 2] - a[:, :, 1]) / 1e3)
show("first polynomial lands (2 -> 3)", (a[:, :, 3] - a[:, :, 2]) / 1e3)
show("first polynomial transformed (3 -> 4)", (a[:, :, 4] - a[:, :, 3]) / 1e3)
show("remaining polynomials (4 -> 5)", (a[:, :, 5] - a[:, :, 4]) / 1e3)
show("exit after the first entry", rel(5))
print(f"launch span (first entry -> last exit): {(a[:, :, 5].max() - t0) / 1e3:.2f} us; "
      f"previous last exit -> this last exit: {(a[:, :, 5].max() - a[:, :, 7].max()) / 1e3:.2f} us")
