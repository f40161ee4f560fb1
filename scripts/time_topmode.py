"""Step time per top-interpolation mode: python scripts/time_topmode.py [C]  (C in 1..3, default 2)"""
import json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch, synth
import paper_1602_02740_b200 as tg
cfg = int(sys.argv[1]) if len(sys.argv) > 1 else 2
u, v = synth.config_inputs(cfg)
u, v = torch.from_numpy(u).cuda(), torch.from_numpy(v).cuda()
B = {1: 3, 2: 4, 3: 8}[cfg]
kw = {1: dict(t4=10**9, t3=10**9), 2: dict(t4=32, t3=32), 3: {}}[cfg]
ref = None
for mode in (2, 4, 3, 1, 0):
    tg.set_top_stream(mode)
    w = tg.toom_mul_batched(u, v, B=B, **kw)
    torch.cuda.synchronize()
    ref = w.clone() if ref is None else ref
    same = bool(torch.equal(w, ref))
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(10):
        tg.toom_mul_batched(u, v, B=B, out=w, **kw)
    e1.record(); torch.cuda.synchronize()
    tg.profile_enable(True); tg.toom_mul_batched(u, v, B=B, out=w, **kw); prof = tg.profile_collect(); tg.profile_enable(False)
    print(json.dumps({"config": cfg, "mode": mode, "ms": e0.elapsed_time(e1) / 10, "same": same, "interp_ms": prof["interp"]["ms"], "base_ms": prof["base"]["ms"]}))
