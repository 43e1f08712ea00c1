"""256 x 2^16 Goldilocks: the four-step (dif / dit) against the six-step 2^8 x 2^8 through the column passes."""
import os, sys
import numpy as np, torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2405_11353_b200 as P
GOLD = (1 << 64) - (1 << 32) + 1
L = int(sys.argv[1]) if len(sys.argv) > 1 else 16
B = (1 << 24) >> L
params = P.FieldParams(GOLD, 7, 64)
x = torch.from_numpy(np.random.default_rng(1).integers(0, GOLD, size=(B, 1 << L), dtype=np.uint64).view(np.int64)).view(torch.uint64).cuda()
y = torch.empty_like(x)
s = torch.cuda.current_stream().cuda_stream
ref = None
for variant, n1 in (("dif", None), ("dit", None), ("pease_nc", None), ("sixstep", 1 << ((L + 1) // 2))):
    plan = P.make_plan(params, variant, 1 << L, n1=n1) if variant == "sixstep" else P.make_plan(params, variant, 1 << L)
    dp = P.algorithms.device_plan_for(plan, 8, 0)
    for _ in range(3): dp.exec_device(x.data_ptr(), y.data_ptr(), B, False, s)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(20): dp.exec_device(x.data_ptr(), y.data_ptr(), B, False, s)
    e1.record(); torch.cuda.synchronize()
    if ref is None: ref = y.clone()
    print(f"{B} x 2^{L} {variant:9s} {e0.elapsed_time(e1) / 20 * 1000:8.1f} us/step  same output: {bool(torch.equal(y.view(torch.int64), ref.view(torch.int64)))}")
