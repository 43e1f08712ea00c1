"""Is the config-2 step loop CPU-launch bound?  Times K back-to-back device
calls (a) with per-step events as bench.py does, (b) without, (c) replayed
from a CUDA graph, all over rotating buffers > L2."""
import os, sys, time
import numpy as np, torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2405_11353_b200 as P
from paper_2405_11353_b200.configs import CONFIGS, seeded_input
cfg, variant = int(sys.argv[1]), sys.argv[2]
K = 200
w = CONFIGS[cfg]
plan = P.make_plan(P.FieldParams(w.p, w.g, w.w), variant, w.n, n1=w.n1)
dp = P.algorithms.device_plan_for(plan, w.word, 0)
tdt = torch.uint32 if w.word == 4 else torch.uint64
x0 = torch.from_numpy(seeded_input(w).view(np.int32 if w.word == 4 else np.int64)).view(tdt).cuda()
nset = 4
xs = [x0.clone() for _ in range(nset)]
ys = [torch.empty_like(x0) for _ in range(nset)]
st = torch.cuda.Stream()
s = st.cuda_stream
def loop(ev):
    for i in range(K):
        if ev: ev[i][0].record(st)
        dp.exec_device(xs[i % nset].data_ptr(), ys[i % nset].data_ptr(), w.batch, False, s)
        if ev: ev[i][1].record(st)
with torch.cuda.stream(st):
    for _ in range(5): loop(None)
    torch.cuda.synchronize()
    for mode in ("events", "plain"):
        evs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(K)] if mode == "events" else None
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        e0.record(st); loop(evs); e1.record(st)
        t1 = time.perf_counter()
        torch.cuda.synchronize()
        per = np.mean([a.elapsed_time(b) for a, b in evs]) * 1e3 if evs else float("nan")
        print(f"{mode:7s}: total {e0.elapsed_time(e1)/K*1e3:.1f} us/step, per-launch events {per:.1f} us, CPU enqueue {(t1-t0)/K*1e6:.1f} us/step")
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g, stream=st):
        loop(None)
    g.replay(); torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(st); g.replay(); e1.record(st); torch.cuda.synchronize()
    print(f"graph  : total {e0.elapsed_time(e1)/K*1e3:.1f} us/step")
