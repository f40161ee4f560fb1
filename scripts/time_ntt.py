"""Time the Toom top level over the NTT inner multiplier (toom_mul_ntt) on the
C4 / C5 operands: python scripts/time_ntt.py C B [reps]"""
import json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch, synth
import paper_1602_02740_b200 as tg
cfg, B = int(sys.argv[1]), int(sys.argv[2])
reps = int(sys.argv[3]) if len(sys.argv) > 3 else 3
u, v = synth.config_inputs(cfg)
u, v = torch.from_numpy(u).cuda(), torch.from_numpy(v).cuda()
w = tg.toom_mul_ntt(u, v, B=B); torch.cuda.synchronize()
ref = tg.toom_mul(u, v, B={4: 4, 5: 16}[cfg]); torch.cuda.synchronize()
same = bool(torch.equal(w, ref))
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(reps):
    tg.toom_mul_ntt(u, v, B=B, out=w)
e1.record(); torch.cuda.synchronize()
print(json.dumps({"config": cfg, "B": B, "ms": e0.elapsed_time(e1) / reps, "equal_to_toom_path": same,
                  "launches": tg.last_launch_count()}))
