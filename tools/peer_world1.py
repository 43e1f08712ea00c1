"""DistributedSixStep(exchange="peer") in a one-rank NCCL group: exercises the
symmetric-memory plumbing (rendezvous, buffer_ptrs, barriers) around the fused
pack-to-peer kernel.  Writes the input and the output of the last of three
calls to argv[1] (.npz) and prints one JSON line; tests/test_gpu_parity.py
runs it in a subprocess with a timeout and checks the output against the oracle."""
import json, os, sys
import numpy as np
import torch
import torch.distributed as dist
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2405_11353_b200 as P
from paper_2405_11353_b200.distributed import DistributedSixStep, column_slab, assemble_output

GOLD = 2**64 - 2**32 + 1
os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
os.environ.setdefault("MASTER_PORT", str(29000 + os.getpid() % 1000))
torch.cuda.set_device(0)
dist.init_process_group("nccl", rank=0, world_size=1, device_id=torch.device("cuda:0"))
res = {}
try:
    n, n1 = 1 << 18, 1 << 9
    x = np.random.default_rng(57).integers(0, GOLD, size=n, dtype=np.uint64)
    ds = DistributedSixStep(P.FieldParams(GOLD, 7, 64), n, n1=n1, exchange="peer")
    slab = torch.from_numpy(column_slab(x, 0, 1, ds.n1, ds.n2).view(np.int64)).view(torch.uint64).cuda()
    outs = []
    for _ in range(3):       # reuse of the symmetric receive buffer across calls
        outs.append(ds.run(slab).cpu().view(torch.int64).numpy().view(np.uint64).copy())
    got = assemble_output([outs[-1]], ds.n1, ds.n2)
    np.savez(sys.argv[1], x=x, out=got)
    res = {"ok": bool(all(np.array_equal(o, outs[0]) for o in outs)), "n": n, "n1": n1}
except Exception as exc:
    res = {"ok": False, "error": repr(exc)[:400]}
finally:
    dist.destroy_process_group()
print(json.dumps(res), flush=True)
