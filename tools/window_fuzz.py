"""Randomised dependency patterns for the launch window (NTT_FLAG_INDEPENDENT): random
(src, dst, direction) single-pass launches over a small pool of device buffers -- chains,
in-place, write-after-read, write-after-write, different batch sizes (exclusive and
non-exclusive grids), a multi-pass launch now and then -- enqueued without any host sync and
replayed sequentially on the CPU oracle.  python tools/window_fuzz.py [rounds] [seed]"""
import os, random, sys
import numpy as np, torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2405_11353_b200 as P
from oracle import oracle as O
p, g, L, B = 998244353, 3, 12, 1536
rounds = int(sys.argv[1]) if len(sys.argv) > 1 else 20
rng = random.Random(int(sys.argv[2]) if len(sys.argv) > 2 else 1)
params = P.FieldParams(p, g)
plans = {}
for v in ("pease_nc", "dit", "dif", "stockham"):
    plans[(v, False)] = P.algorithms.device_plan_for(P.make_plan(params, v, 1 << L), 4, 0)
    plans[(v, True)] = P.algorithms.device_plan_for(P.make_plan(params, v, 1 << L, P.INVERSE), 4, 0)
big = P.algorithms.device_plan_for(P.make_plan(params, "pease_nc", 1 << 15), 4, 0)      # multi-pass: ends a run
NB = 5
st = torch.cuda.Stream()
bad = 0
for r in range(rounds):
    host = [np.random.default_rng(100 * r + i).integers(0, p, size=(B, 1 << L), dtype=np.uint64).astype(np.uint32) for i in range(NB)]
    with torch.cuda.stream(st):
        dev = [torch.from_numpy(h.view(np.int32)).view(torch.uint32).cuda() for h in host]
        bx = torch.zeros((8, 1 << 15), dtype=torch.int32, device="cuda").view(torch.uint32)
        st.synchronize()
        ops = []
        for _ in range(rng.randint(8, 30)):
            s, d = rng.randrange(NB), rng.randrange(NB)
            v, inv = rng.choice(("pease_nc", "dit", "dif", "stockham")), rng.random() < 0.4
            rows = rng.choice((B, B, 640, 200))            # 640 / 200 rows: grids that do not fill the machine
            if rng.random() < 0.1:
                big.exec_device(bx.data_ptr(), bx.data_ptr(), 8, False, st.cuda_stream)
            plans[(v, inv)].exec_device(dev[s].data_ptr(), dev[d].data_ptr(), rows, inv, st.cuda_stream, independent=True)
            ops.append((s, d, v, inv, rows))
        st.synchronize()
    for s, d, v, inv, rows in ops:
        out = O.ntt(host[s][:rows], p, g, 32, v, inverse=inv, scale=inv)
        host[d] = host[d].copy()
        host[d][:rows] = out
    for i in range(NB):
        got = dev[i].cpu().view(torch.int32).numpy().view(np.uint32)
        if not np.array_equal(got, host[i]):
            bad += 1
            print(f"round {r}: buffer {i} differs; ops = {ops}")
print(f"{rounds} rounds, {bad} mismatching buffers")
