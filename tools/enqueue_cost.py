"""CPU cost of enqueueing pinned async copies and transforms (host-side
bottleneck check for ntt_exec_host's chunked pipeline)."""
import os, sys, time
import numpy as np, torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2405_11353_b200 as P
from paper_2405_11353_b200.configs import CONFIGS, seeded_input
w = CONFIGS[2]
plan = P.make_plan(P.FieldParams(w.p, w.g, w.w), "pease_nc", w.n)
dp = P.algorithms.device_plan_for(plan, w.word, 0)
hin = torch.from_numpy(seeded_input(w).view(np.int32)).pin_memory()
d = torch.empty_like(hin, device="cuda")
s = torch.cuda.Stream()
for chunks in (8, 32):
    rows = w.batch // chunks
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    with torch.cuda.stream(s):
        for c in range(chunks):
            d[c * rows:(c + 1) * rows].copy_(hin[c * rows:(c + 1) * rows], non_blocking=True)
    t1 = time.perf_counter()
    for c in range(chunks):
        dp.exec_device(d[c * rows:].data_ptr(), d[c * rows:].data_ptr(), rows, False, s.cuda_stream)
    t2 = time.perf_counter()
    torch.cuda.synchronize()
    print(f"chunks={chunks}: copy enqueue {(t1-t0)/chunks*1e6:.1f} us each, transform enqueue {(t2-t1)/chunks*1e6:.1f} us each")
# host exec call end-to-end breakdown
for _ in range(3): dp.exec_host(hin.data_ptr(), hin.data_ptr(), w.batch, False, 0)
t0 = time.perf_counter()
for _ in range(10): dp.exec_host(hin.data_ptr(), hin.data_ptr(), w.batch, False, 0)
print(f"exec_host: {(time.perf_counter()-t0)/10*1e3:.3f} ms")
