"""Steady-state DRAM traffic per launch of one workload: K back-to-back
launches (rotating input/output sets > L2) inside a cudaProfilerStart/Stop
range, for `ncu --replay-mode range` (a single-launch capture under-reads the
writes still sitting in L2 when the launch ends).
    ncu --replay-mode app-range --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum \
        python tools/traffic_range.py CFG VARIANT [K]"""
import os, sys
import numpy as np, torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2405_11353_b200 as P
from paper_2405_11353_b200.configs import CONFIGS, seeded_input
cfg, variant = int(sys.argv[1]), sys.argv[2]
K = int(sys.argv[3]) if len(sys.argv) > 3 else 16
w = CONFIGS[cfg]
plan = P.make_plan(P.FieldParams(w.p, w.g, w.w), variant, w.n, n1=w.n1)
dp = P.algorithms.device_plan_for(plan, w.word, 0)
tdt = torch.uint32 if w.word == 4 else torch.uint64
x0 = torch.from_numpy(seeded_input(w).view(np.int32 if w.word == 4 else np.int64)).view(tdt).cuda()
nset = max(2, int(np.ceil(3 * 126e6 / (2 * x0.numel() * w.word))) + 1)
xs = [x0] + [x0.clone() for _ in range(nset - 1)]
ys = [torch.empty_like(x0) for _ in range(nset)]
s = torch.cuda.current_stream().cuda_stream
for i in range(3):
    dp.exec_device(xs[i % nset].data_ptr(), ys[i % nset].data_ptr(), w.batch, False, s)
torch.cuda.synchronize()
torch.cuda.cudart().cudaProfilerStart()
for i in range(K):
    dp.exec_device(xs[i % nset].data_ptr(), ys[i % nset].data_ptr(), w.batch, False, s)
torch.cuda.synchronize()
torch.cuda.cudart().cudaProfilerStop()
print(f"ranged {K} steps of config {cfg} {variant}, {nset} buffer sets")
