"""Host <-> device copy bandwidth with pinned memory: each direction alone and both at once
(the bound of the pipelined fqnm_step_host, which moves the state in and out every call)."""
import json
import time
import torch

n = 1 << 30                                   # 4 GiB of int32 each way
h_in = torch.empty(n, dtype=torch.int32, pin_memory=True)
h_out = torch.empty(n, dtype=torch.int32, pin_memory=True)
d_in = torch.empty(n, dtype=torch.int32, device="cuda")
d_out = torch.zeros(n, dtype=torch.int32, device="cuda")
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()


def run(h2d, d2h):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    if h2d:
        with torch.cuda.stream(s1):
            d_in.copy_(h_in, non_blocking=True)
    if d2h:
        with torch.cuda.stream(s2):
            h_out.copy_(d_out, non_blocking=True)
    torch.cuda.synchronize()
    return time.perf_counter() - t0


for _ in range(2):
    run(True, True)
res = {"bytes_each_way": 4 * n,
       "h2d_alone_gbs": 4 * n / min(run(True, False) for _ in range(3)) / 1e9,
       "d2h_alone_gbs": 4 * n / min(run(False, True) for _ in range(3)) / 1e9}
t = min(run(True, True) for _ in range(3))
res["both_seconds"] = t
res["both_each_way_gbs"] = 4 * n / t / 1e9
print(json.dumps(res))
