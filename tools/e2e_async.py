"""Host-buffer throughput of config 2 through ntt_exec_host, synchronous vs
NTT_FLAG_HOST_ASYNC (steps pipelined): python tools/e2e_async.py [steps]
(the chunk counts are fixed in ntt_exec_host: 8 synchronous, 2 asynchronous; the sweep that chose them
used an NTT_HOST_CHUNKS override that has since been removed)."""
import os, sys, time
import numpy as np, torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2405_11353_b200 as P
from paper_2405_11353_b200.configs import CONFIGS, seeded_input
steps = int(sys.argv[1]) if len(sys.argv) > 1 else 20
w = CONFIGS[2]
dp = P.algorithms.device_plan_for(P.make_plan(P.FieldParams(w.p, w.g, w.w), "pease_nc", w.n), 4, 0)
hin = torch.from_numpy(seeded_input(w).view(np.int32)).pin_memory()
hout = torch.empty_like(hin).pin_memory()
st = torch.cuda.Stream()
for asyn in (False, True):
    for _ in range(3):
        dp.exec_host(hin.data_ptr(), hout.data_ptr(), w.batch, False, st.cuda_stream, asyn)
    st.synchronize()
    t0 = time.perf_counter()
    for _ in range(steps):
        dp.exec_host(hin.data_ptr(), hout.data_ptr(), w.batch, False, st.cuda_stream, asyn)
    st.synchronize()
    dt = (time.perf_counter() - t0) / steps
    print(f"chunks={os.environ.get('NTT_HOST_CHUNKS', 'default')} async={asyn}: {dt*1e3:.3f} ms/step "
          f"{w.batch/dt/1e6:.3f} M NTT/s")
