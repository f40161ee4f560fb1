"""PCIe copy rates with pinned host buffers (e2e context): H2D, D2H, both at once."""
import json, torch
n = 134217728 // 4
h1 = torch.empty(n, dtype=torch.uint32).pin_memory(); h2 = torch.empty(n, dtype=torch.uint32).pin_memory()
d1 = torch.empty(n, dtype=torch.uint32, device="cuda"); d2 = torch.empty(n, dtype=torch.uint32, device="cuda")
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
def t(f, reps=5):
    f(); torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps): f()
    torch.cuda.synchronize(); e1.record(); torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps
def both():
    with torch.cuda.stream(s1): d1.copy_(h1, non_blocking=True)
    with torch.cuda.stream(s2): h2.copy_(d2, non_blocking=True)
    torch.cuda.current_stream().wait_stream(s1); torch.cuda.current_stream().wait_stream(s2)
r = {"h2d_ms": t(lambda: d1.copy_(h1, non_blocking=True)), "d2h_ms": t(lambda: h2.copy_(d2, non_blocking=True)), "both_ms": t(both)}
r.update({k.replace("_ms", "_GBps"): 134217728 / (v * 1e-3) / 1e9 for k, v in r.items()})
print(json.dumps(r))
