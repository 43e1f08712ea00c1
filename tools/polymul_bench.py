"""Polynomial products c = a * b mod (x^N - 1) (polymul.cyclic_mul_ntt): the
fused device path (forward of both operands in one launch + ntt_exec_pointwise_inverse)
vs the three-call path (forward, pointwise kernel, intt); CUDA events, graph replay.
    python tools/polymul_bench.py [L] [batch]"""
import os, sys
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2405_11353_b200 as P

L = int(sys.argv[1]) if len(sys.argv) > 1 else 12
B = int(sys.argv[2]) if len(sys.argv) > 2 else 4096
p, n = 998244353, 1 << L
params = P.FieldParams(p, 3)
fwd = P.algorithms._device_plan(params, n, "pease_nc", P.FORWARD, None, None, 4, 0)
inv = P.algorithms._device_plan(params, n, "pease_nc", P.INVERSE, None, None, 4, 0)
ab = torch.randint(0, p, (2, B, n), dtype=torch.int64, device="cuda").to(torch.int32).view(torch.uint32)
spec = torch.empty_like(ab)
prod = torch.empty_like(ab[0])
out = torch.empty_like(ab[0])
st = torch.cuda.Stream()
s = st.cuda_stream


def fused():
    fwd.exec_device(ab.data_ptr(), spec.data_ptr(), 2 * B, False, s)
    inv.pointwise_inverse(spec[0].data_ptr(), spec[1].data_ptr(), out.data_ptr(), B, s)


def three():
    fwd.exec_device(ab.data_ptr(), spec.data_ptr(), 2 * B, False, s)
    inv.pointwise(spec[0].data_ptr(), spec[1].data_ptr(), prod.data_ptr(), B * n, s)
    inv.exec_device(prod.data_ptr(), out.data_ptr(), B, True, s)


res = {}
for name, fn in (("fused", fused), ("three_calls", three)):
    with torch.cuda.stream(st):
        for _ in range(3):
            fn()
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g, stream=st):
            for _ in range(20):
                fn()
        g.replay()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(st); g.replay(); e1.record(st)
    torch.cuda.synchronize()
    t = e0.elapsed_time(e1) / 20 * 1e-3
    res[name] = out.clone()
    print(f"{name:12s} 2^{L} x {B}: {t*1e6:8.1f} us/step  {B/t/1e6:8.2f} M products/s  "
          f"(algorithmic {3*B*n*4/t/1e9:7.1f} GB/s: read a, b + write c)")
print("agree:", bool(torch.equal(res["fused"], res["three_calls"])))
