"""Time one BASELINE config (CUDA events, device-resident) and check its full
output SHA-256 against the reference's: python tools/time_hash.py CFG VARIANT [STEPS]"""
import hashlib, os, sys
import numpy as np, torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2405_11353_b200 as P
from paper_2405_11353_b200.configs import CONFIGS, GOLDEN, seeded_input
cfg, variant = int(sys.argv[1]), sys.argv[2]
steps = int(sys.argv[3]) if len(sys.argv) > 3 else 10
w = CONFIGS[cfg]
plan = P.make_plan(P.FieldParams(w.p, w.g, w.w), variant, w.n, n1=w.n1)
dp = P.algorithms.device_plan_for(plan, w.word, 0)
sdt = torch.int32 if w.word == 4 else torch.int64
x = torch.from_numpy(seeded_input(w).view(np.int32 if w.word == 4 else np.int64)).cuda()
y = torch.empty_like(x)
s = torch.cuda.current_stream().cuda_stream
dp.exec_device(x.data_ptr(), y.data_ptr(), w.batch, False, s)
torch.cuda.synchronize()
h = hashlib.sha256(y.cpu().numpy().astype("<i4" if w.word == 4 else "<i8").tobytes()).hexdigest()
for _ in range(3): dp.exec_device(x.data_ptr(), y.data_ptr(), w.batch, False, s)
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(steps): dp.exec_device(x.data_ptr(), y.data_ptr(), w.batch, False, s)
e1.record(); torch.cuda.synchronize()
print(f"cfg{cfg} {variant} lib={os.path.basename(os.environ.get('NTT_LIB_PATH') or 'base')}: "
      f"{e0.elapsed_time(e1)/steps*1000:.1f} us/step sha_ok={h == GOLDEN[cfg][1]}")
