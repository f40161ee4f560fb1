"""C2 timing vs chunk size (L2 residency of the intermediates):
python scripts/time_c2_chunks.py"""
import json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch, synth
import paper_1602_02740_b200 as tg
u, v = synth.config_inputs(2)
u, v = torch.from_numpy(u).cuda(), torch.from_numpy(v).cuda()
ref = tg.toom_mul_batched(u, v, B=4, t4=32, t3=32); torch.cuda.synchronize()
for chunk in [0, 32768, 16384, 8192, 4096, 2048]:
    out = torch.empty_like(ref)
    tg.toom_mul_batched(u, v, B=4, t4=32, t3=32, chunk=chunk, out=out); torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(10):
        tg.toom_mul_batched(u, v, B=4, t4=32, t3=32, chunk=chunk, out=out)
    e1.record(); torch.cuda.synchronize()
    tg.profile_enable(True); tg.toom_mul_batched(u, v, B=4, t4=32, t3=32, chunk=chunk, out=out); prof = tg.profile_collect(); tg.profile_enable(False)
    print(json.dumps({"chunk": chunk, "ms": e0.elapsed_time(e1) / 10, "equal": bool(torch.equal(out, ref)),
                      "prof": {k: round(x["ms"], 4) for k, x in prof.items()}}), flush=True)
