"""Time one config through the public API (CUDA events) and print the per-stage
profile: python scripts/time_cfg.py C [reps]   (C in 1..5)"""
import json, os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch, synth
import paper_1602_02740_b200 as tg
cfg = int(sys.argv[1]); reps = int(sys.argv[2]) if len(sys.argv) > 2 else 3
u, v = synth.config_inputs(cfg)
u, v = torch.from_numpy(u).cuda(), torch.from_numpy(v).cuda()
B = {1: 3, 2: 4, 3: 8, 4: 4, 5: 16}[cfg]
kw = {1: dict(t4=10**9, t3=10**9), 2: dict(t4=32, t3=32), 3: {}, 4: {}, 5: {}}[cfg]
def run():
    if cfg >= 4:
        return tg.toom_mul(u, v, B=B)
    return tg.toom_mul_batched(u, v, B=B, **kw)
run(); torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
t0 = time.perf_counter()
e0.record()
for _ in range(reps):
    run()
e1.record(); torch.cuda.synchronize()
wall = (time.perf_counter() - t0) / reps * 1e3
ms = e0.elapsed_time(e1) / reps
tg.profile_enable(True); run(); prof = tg.profile_collect(); tg.profile_enable(False)
print(json.dumps({"config": cfg, "ms": ms, "wall_ms": wall, "launches": tg.last_launch_count(), "prof": prof}))
