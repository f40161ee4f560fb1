"""C2 step time per top-interpolation mode: python scripts/time_topmode.py"""
import json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch, synth
import paper_1602_02740_b200 as tg
u, v = synth.config_inputs(2)
u, v = torch.from_numpy(u).cuda(), torch.from_numpy(v).cuda()
ref = None
for mode in (2, 4, 3, 1, 0):
    tg.set_top_stream(mode)
    w = tg.toom_mul_batched(u, v, B=4, t4=32, t3=32)
    torch.cuda.synchronize()
    ref = w.clone() if ref is None else ref
    same = bool(torch.equal(w, ref))
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(10):
        tg.toom_mul_batched(u, v, B=4, t4=32, t3=32, out=w)
    e1.record(); torch.cuda.synchronize()
    tg.profile_enable(True); tg.toom_mul_batched(u, v, B=4, t4=32, t3=32, out=w); prof = tg.profile_collect(); tg.profile_enable(False)
    print(json.dumps({"mode": mode, "ms": e0.elapsed_time(e1) / 10, "same": same, "interp_ms": prof["interp"]["ms"], "base_ms": prof["base"]["ms"]}))
