"""Experiment: config 4 (512 x 2^20 u32 Pease_nc) executed as sub-batches of C
polynomials, so that each sub-batch's pass-0 intermediate (C x 4 MiB) can stay
L2-resident between the two pass launches.  Graph-captured, CUDA-event timed.
    python tools/chunk_exp.py [C ...]"""
import os, sys
import numpy as np, torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2405_11353_b200 as P
from paper_2405_11353_b200.configs import CONFIGS, seeded_input

w = CONFIGS[4]
plan = P.make_plan(P.FieldParams(w.p, w.g, w.w), "pease_nc", w.n)
dp = P.algorithms.device_plan_for(plan, w.word, 0)
x = torch.from_numpy(seeded_input(w).view(np.int32)).view(torch.uint32).cuda()
y = torch.empty_like(x)
ref = None
N = w.n
for C in [int(a) for a in sys.argv[1:]] or [512, 64, 32, 16, 8, 4]:
    stream = torch.cuda.Stream()
    def step():
        s = stream.cuda_stream
        for c0 in range(0, w.batch, C):
            dp.exec_device(x.data_ptr() + c0 * N * 4, y.data_ptr() + c0 * N * 4, C, False, s)
    with torch.cuda.stream(stream):
        step(); step()
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g, stream=stream):
        step()
    g.replay(); torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    reps = 10
    with torch.cuda.stream(stream):
        e0.record()
        for _ in range(reps): g.replay()
        e1.record()
    torch.cuda.synchronize()
    h = int(y.view(torch.int32).sum().item())
    if ref is None: ref = h
    print(f"C={C}: {e0.elapsed_time(e1)/reps*1000:.1f} us/step  ok={h == ref}", flush=True)
