"""K2 vs K2P timing on a cfg3-sized problem (diagnostic for the persistent stepper)."""
import os
import sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2604_06947_b200 as F
import workloads as W
n = 1 << 24
q0 = torch.tensor(W.q0_cfg3(n), dtype=torch.int32, device="cuda")
for kern, steps in ((2, 1024), (12, 1024), (2, 10000), (12, 10000)):
    p = F.fqnm_plan(n, 1e-6, 0.5, F.LINEAR, F.PERIODIC)
    F.fqnm_debug_override(p, kern)
    q = q0.clone()
    F.fqnm_step(p, q, steps)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    F.fqnm_step(p, q, steps)
    e1.record()
    torch.cuda.synchronize()
    print(os.environ.get("FQNM_LIBPATH", "default")[-30:], kern, steps, round(e0.elapsed_time(e1), 3))
