import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
os.environ["RFGPU_DEBUG_PTR"] = "1"
import numpy as np
variant = sys.argv[1]
import paper_1607_01649_b200 as rf
if variant == "noop":
    fn = lambda b: None
elif variant == "torch":
    import torch
    fn = lambda b: torch.from_numpy(b).mul_(1.0)
else:
    import torch, torch.distributed as dist
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT="29555")
    dist.init_process_group("gloo", rank=0, world_size=1)
    fn = lambda b: dist.all_reduce(torch.from_numpy(b))
ctx = rf.Context(0, 0, 2, host_sum=fn)
a = np.asfortranarray(np.random.default_rng(0).standard_normal((300, 200)))
dm = rf.DeviceMatrix.upload(ctx, a)
try:
    rf.rsvd(dm, 10, 5, 1, 1, reorthonormalize=True)
    print(variant, "rsvd ok", flush=True)
except Exception as e:
    print(variant, "rsvd failed", e, flush=True)
