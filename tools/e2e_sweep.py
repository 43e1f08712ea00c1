"""e2e (host buffers through ntt_exec_host) vs chunk count: python tools/e2e_sweep.py CFG VARIANT"""
import os, subprocess, sys
if len(sys.argv) > 3:
    import time
    import numpy as np, torch
    sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
    import paper_2405_11353_b200 as P
    from paper_2405_11353_b200.configs import CONFIGS, seeded_input
    w = CONFIGS[int(sys.argv[1])]
    plan = P.make_plan(P.FieldParams(w.p, w.g, w.w), sys.argv[2], w.n, n1=w.n1)
    dp = P.algorithms.device_plan_for(plan, w.word, 0)
    x = seeded_input(w)
    hin = torch.from_numpy(x.view(np.int32 if w.word == 4 else np.int64)).pin_memory()
    hout = torch.empty_like(hin).pin_memory()
    s = torch.cuda.current_stream().cuda_stream
    for _ in range(3): dp.exec_host(hin.data_ptr(), hout.data_ptr(), w.batch, False, s)
    K = 20
    t0 = time.perf_counter()
    for _ in range(K): dp.exec_host(hin.data_ptr(), hout.data_ptr(), w.batch, False, s)
    dt = (time.perf_counter() - t0) / K
    print(f"chunks={os.environ.get('NTT_HOST_CHUNKS', 'default'):>7}: {dt*1e3:.3f} ms/step  {w.batch/dt/1e6:.3f} M NTT/s")
else:
    for c in ("0", "4", "8", "16", "32", "64"):
        env = dict(os.environ, NTT_HOST_CHUNKS=c)
        subprocess.run([sys.executable, __file__, sys.argv[1], sys.argv[2], "run"], env=env)
