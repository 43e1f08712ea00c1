"""Run a batched u32 transform of size 2^L a few times (for ncu): python tools/prof_L.py L [variant] [iters]"""
import os, sys
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2405_11353_b200 as P
L = int(sys.argv[1]); variant = sys.argv[2] if len(sys.argv) > 2 else "pease_nc"
iters = int(sys.argv[3]) if len(sys.argv) > 3 else 3
p = 998244353; n = 1 << L; B = (1 << 28) // n
plan = P.make_plan(P.FieldParams(p, 3), variant, n)
dp = P.algorithms.device_plan_for(plan, 4, 0)
x = torch.randint(0, p, (B, n), dtype=torch.int64, device="cuda").to(torch.int32).view(torch.uint32)
y = torch.empty_like(x)
s = torch.cuda.current_stream().cuda_stream
for _ in range(iters):
    dp.exec_device(x.data_ptr(), y.data_ptr(), B, False, s)
torch.cuda.synchronize()
print("ok", L, variant)
