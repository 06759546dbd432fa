"""Host<->device copy bandwidth with pinned memory: H2D alone, D2H alone, both at once (context for e2e)."""
import json
import torch
n = 268435456
h1 = torch.empty(n, dtype=torch.float64).pin_memory()
h2 = torch.empty(n, dtype=torch.float64).pin_memory()
d1 = torch.empty(n, dtype=torch.float64, device="cuda")
d2 = torch.empty(n, dtype=torch.float64, device="cuda")
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
def t(fn):
    torch.cuda.synchronize(); e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
    e0.record(); fn(); e1.record(); torch.cuda.synchronize(); return e0.elapsed_time(e1) * 1e-3
for _ in range(2):
    d1.copy_(h1, non_blocking=True); h2.copy_(d2, non_blocking=True)
th = t(lambda: d1.copy_(h1, non_blocking=True))
td = t(lambda: h2.copy_(d2, non_blocking=True))
def both():
    with torch.cuda.stream(s1): d1.copy_(h1, non_blocking=True)
    with torch.cuda.stream(s2): h2.copy_(d2, non_blocking=True)
    torch.cuda.current_stream().wait_stream(s1); torch.cuda.current_stream().wait_stream(s2)
tb = t(both)
B = n * 8
print(json.dumps({"h2d_gbs": B / th / 1e9, "d2h_gbs": B / td / 1e9, "both_ms": tb * 1e3, "both_gbs_each": B / tb / 1e9,
                  "bytes": B}))
