"""Time the rank-local steps of the distributed four-step on ONE GPU for a
world size G (step A and step B of one rank, the all-to-all excluded):
    python tools/dist_emul_time.py G"""
import os, sys
import numpy as np, torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2405_11353_b200 as P
from paper_2405_11353_b200.configs import CONFIGS
G = int(sys.argv[1]) if len(sys.argv) > 1 else 1
w = CONFIGS[5]
plan = P.make_plan(P.FieldParams(w.p, w.g, w.w), "sixstep", w.n, n1=w.n1)
dp = P.algorithms.device_plan_for(plan, 8, 0)
n_local = w.n // G
x = torch.randint(0, 2**62, (n_local,), dtype=torch.int64, device="cuda").view(torch.uint64)
y = torch.empty_like(x)
s = torch.cuda.current_stream().cuda_stream
for step in (0, 1):
    for _ in range(2): dp.sixstep_dist_step(step, 0, G, x.data_ptr(), y.data_ptr(), s)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(5): dp.sixstep_dist_step(step, 0, G, x.data_ptr(), y.data_ptr(), s)
    e1.record(); torch.cuda.synchronize()
    print(f"G={G} step {'AB'[step]}: {e0.elapsed_time(e1)/5*1000:.1f} us per rank")
