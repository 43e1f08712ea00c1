"""Batched u32 NTT sweep N = 2^12 .. 2^20 (P = 998244353, 1 GiB of residues per
step, CUDA-graph replay, CUDA events): NTT/s and fraction of the HBM roofline.
    python tools/sweep.py [variant] [Lmin] [Lmax]"""
import json, os, sys
import numpy as np, torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2405_11353_b200 as P

variant = sys.argv[1] if len(sys.argv) > 1 else "pease_nc"
lmin = int(sys.argv[2]) if len(sys.argv) > 2 else 12
lmax = int(sys.argv[3]) if len(sys.argv) > 3 else 20
peak = json.load(open(os.path.join(os.path.dirname(__file__), "..", "MEASURED_PEAKS.json")))["hbm_gbs"] \
    if os.path.exists(os.path.join(os.path.dirname(__file__), "..", "MEASURED_PEAKS.json")) else 6550.0
p, g = 998244353, 3
total = 1 << 28                       # residues per step (1 GiB)
params = P.FieldParams(p, g)
for L in range(lmin, lmax + 1):
    n = 1 << L
    B = total // n
    plan = P.make_plan(params, variant, n)
    dp = P.algorithms.device_plan_for(plan, 4, 0)
    x = torch.randint(0, p, (B, n), dtype=torch.int64, device="cuda").to(torch.int32).view(torch.uint32)
    y = torch.empty_like(x)
    st = torch.cuda.Stream()
    with torch.cuda.stream(st):
        for _ in range(3):
            dp.exec_device(x.data_ptr(), y.data_ptr(), B, False, st.cuda_stream)
    torch.cuda.synchronize()
    reps = 10
    gph = torch.cuda.CUDAGraph()
    with torch.cuda.graph(gph, stream=st):
        for _ in range(reps):
            dp.exec_device(x.data_ptr(), y.data_ptr(), B, False, st.cuda_stream)
    gph.replay(); torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with torch.cuda.stream(st):
        e0.record(); gph.replay(); e1.record()
    torch.cuda.synchronize()
    t = e0.elapsed_time(e1) / reps * 1e-3
    gbs = 2 * total * 4 / t / 1e9
    print(json.dumps({"L": L, "batch": B, "variant": variant, "ms": round(t * 1e3, 3), "ntt_per_s": B / t,
                      "gbfly_per_s": B * (n // 2) * L / t / 1e9, "alg_gbs": round(gbs, 1),
                      "roofline_frac": round(gbs / peak, 3)}), flush=True)
    del x, y, gph
