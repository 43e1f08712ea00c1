"""Run one workload a few times (for ncu captures): python tools/prof_case.py CFG VARIANT [ITERS] [inv]"""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2405_11353_b200 as P  # noqa: E402
from paper_2405_11353_b200.configs import CONFIGS, seeded_input  # noqa: E402

cfg, variant = int(sys.argv[1]), sys.argv[2]
iters = int(sys.argv[3]) if len(sys.argv) > 3 else 5
inv = len(sys.argv) > 4 and sys.argv[4] == "inv"
w = CONFIGS[cfg]
params = P.FieldParams(w.p, w.g, w.w)
plan = P.make_plan(params, variant, w.n, P.INVERSE if inv else P.FORWARD, n1=w.n1)
dp = P.algorithms.device_plan_for(plan, w.word, 0)
x = seeded_input(w)
tdt = torch.uint32 if w.word == 4 else torch.uint64
xd = torch.from_numpy(x.view(np.int32 if w.word == 4 else np.int64)).view(tdt).cuda()
yd = torch.empty_like(xd)
s = torch.cuda.current_stream().cuda_stream
for _ in range(iters):
    dp.exec_device(xd.data_ptr(), yd.data_ptr(), w.batch, inv, s)
torch.cuda.synchronize()
print("ok", cfg, variant, iters)
