"""K8 variant sweep (FQNM_LIBPATH selects the build): GCUPS on 512^3 EO / linear and a
sha of the state after a fixed run, so variants can be compared for identical output."""
import hashlib
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch
import paper_2604_06947_b200 as F

tag = os.environ.get("TAG", "")
for kind, lam, delta, amp, name in ((F.LINEAR, 0.25, 1e-3, 3000, "linear"),
                                    (F.BURGERS_EO, 1 / 15, 1e-5, 100000, "eo")):
    n = int(os.environ.get("N3", "512"))
    plan = F.fqnm_plan_3d(n, n, n, delta, lam, lam, lam, kind, F.PERIODIC)
    F.fqnm_debug_override(plan, 8)
    g = torch.Generator(device="cuda").manual_seed(0)
    q = torch.randint(-amp, amp, (n, n, n), dtype=torch.int32, device="cuda", generator=g)
    F.fqnm_step(plan, q, 3)
    torch.cuda.synchronize()
    sha = hashlib.sha1(q.cpu().numpy().tobytes()).hexdigest()[:12]
    best = 1e30
    for _ in range(3):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        F.fqnm_step(plan, q, 20)
        e1.record()
        torch.cuda.synchronize()
        best = min(best, e0.elapsed_time(e1))
    print(json.dumps({"tag": tag, "rule": name, "n": n, "GCUPS": round(n ** 3 * 20 / best / 1e6, 1),
                      "sha": sha}), flush=True)
    del plan, q
