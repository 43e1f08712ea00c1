"""Time one batched transform of any field (CUDA events, 1 GiB of u32 / 2 GiB of u64 residues per step):
    python tools/time_field.py P G W LOG2N VARIANT [STEPS]"""
import os, sys
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2405_11353_b200 as P
p, g, w, L, variant = int(sys.argv[1]), int(sys.argv[2]), int(sys.argv[3]), int(sys.argv[4]), sys.argv[5]
steps = int(sys.argv[6]) if len(sys.argv) > 6 else 10
word = 4 if p < (1 << 32) and w <= 32 else 8
n = 1 << L
B = (1 << 28) // n
plan = P.make_plan(P.FieldParams(p, g, w), variant, n)
dp = P.algorithms.device_plan_for(plan, word, 0)
if word == 4:
    x = torch.randint(0, p, (B, n), dtype=torch.int64, device="cuda").to(torch.int32).view(torch.uint32)
else:
    x = torch.randint(0, min(p, (1 << 63) - 1), (B, n), dtype=torch.int64, device="cuda").view(torch.uint64)
y = torch.empty_like(x)
s = torch.cuda.current_stream().cuda_stream
for _ in range(3): dp.exec_device(x.data_ptr(), y.data_ptr(), B, False, s)
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(steps): dp.exec_device(x.data_ptr(), y.data_ptr(), B, False, s)
e1.record(); torch.cuda.synchronize()
print(f"p={p} 2^{L} {variant}: {e0.elapsed_time(e1) / steps * 1000:.1f} us/step ({B} rows)")
