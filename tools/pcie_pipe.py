"""Chunked H2D -> (transform) -> D2H pipeline timings with torch streams, to
separate copy-engine behaviour from the transform: python tools/pcie_pipe.py"""
import os, sys, time
import numpy as np, torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2405_11353_b200 as P
from paper_2405_11353_b200.configs import CONFIGS, seeded_input
w = CONFIGS[2]
plan = P.make_plan(P.FieldParams(w.p, w.g, w.w), "pease_nc", w.n)
dp = P.algorithms.device_plan_for(plan, w.word, 0)
x = seeded_input(w).view(np.int32)
hin = torch.from_numpy(x).pin_memory(); hout = torch.empty_like(hin).pin_memory()
d = torch.empty_like(hin, device="cuda")
sH, sC, sD = torch.cuda.Stream(), torch.cuda.Stream(), torch.cuda.Stream()
def run(chunks, kernel):
    rows = w.batch // chunks
    evs = []
    for c in range(chunks):
        sl = slice(c * rows, (c + 1) * rows)
        with torch.cuda.stream(sH):
            d[sl].copy_(hin[sl], non_blocking=True)
            e = torch.cuda.Event(); e.record(sH)
        sC.wait_event(e)
        if kernel:
            dp.exec_device(d[sl].data_ptr(), d[sl].data_ptr(), rows, False, sC.cuda_stream)
        e2 = torch.cuda.Event(); e2.record(sC); evs.append(e2)
    for c in range(chunks):
        sl = slice(c * rows, (c + 1) * rows)
        sD.wait_event(evs[c])
        with torch.cuda.stream(sD):
            hout[sl].copy_(d[sl], non_blocking=True)
    torch.cuda.synchronize()
for kernel in (False, True):
    for chunks in (1, 4, 8, 16, 32):
        run(chunks, kernel)
        t0 = time.perf_counter()
        for _ in range(10): run(chunks, kernel)
        dt = (time.perf_counter() - t0) / 10
        print(f"kernel={kernel!s:5} chunks={chunks:3d}: {dt*1e3:.3f} ms")

# zero-copy: the transform reads / writes the pinned host buffers directly (UVA)
ref = torch.empty_like(hin)
run(8, True)
ref.copy_(hout)
hout.zero_()
for _ in range(2):
    dp.exec_device(hin.data_ptr(), hout.data_ptr(), w.batch, False, sC.cuda_stream)
torch.cuda.synchronize()
print("zero-copy output equal:", bool(torch.equal(hout, ref)))
t0 = time.perf_counter()
for _ in range(10):
    dp.exec_device(hin.data_ptr(), hout.data_ptr(), w.batch, False, sC.cuda_stream)
torch.cuda.synchronize()
print(f"zero-copy: {(time.perf_counter() - t0) / 10 * 1e3:.3f} ms")

# hybrid: copy engine for H2D, the transform stores straight into pinned host memory
def run_hybrid(chunks):
    rows = w.batch // chunks
    for c in range(chunks):
        sl = slice(c * rows, (c + 1) * rows)
        with torch.cuda.stream(sH):
            d[sl].copy_(hin[sl], non_blocking=True)
            e = torch.cuda.Event(); e.record(sH)
        sC.wait_event(e)
        dp.exec_device(d[sl].data_ptr(), hout[sl].data_ptr(), rows, False, sC.cuda_stream)
    torch.cuda.synchronize()
for chunks in (4, 8, 16):
    hout.zero_()
    run_hybrid(chunks)
    ok = bool(torch.equal(hout, ref))
    t0 = time.perf_counter()
    for _ in range(10): run_hybrid(chunks)
    print(f"hybrid chunks={chunks}: {(time.perf_counter() - t0) / 10 * 1e3:.3f} ms, equal={ok}")
