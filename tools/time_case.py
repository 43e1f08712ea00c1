"""Time one workload (CUDA events, rotating buffers): python tools/time_case.py CFG VARIANT [STEPS]"""
import os, sys
import numpy as np, torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2405_11353_b200 as P
from paper_2405_11353_b200.configs import CONFIGS, seeded_input
cfg, variant = int(sys.argv[1]), sys.argv[2]
steps = int(sys.argv[3]) if len(sys.argv) > 3 else 10
w = CONFIGS[cfg]
plan = P.make_plan(P.FieldParams(w.p, w.g, w.w), variant, w.n, n1=w.n1)
dp = P.algorithms.device_plan_for(plan, w.word, 0)
tdt = torch.uint32 if w.word == 4 else torch.uint64
x = torch.from_numpy(seeded_input(w).view(np.int32 if w.word == 4 else np.int64)).view(tdt).cuda()
y = torch.empty_like(x)
s = torch.cuda.current_stream().cuda_stream
for _ in range(3): dp.exec_device(x.data_ptr(), y.data_ptr(), w.batch, False, s)
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(steps): dp.exec_device(x.data_ptr(), y.data_ptr(), w.batch, False, s)
e1.record(); torch.cuda.synchronize()
print(f"cfg{cfg} {variant}: {e0.elapsed_time(e1)/steps*1000:.1f} us/step")
