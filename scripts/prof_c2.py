"""One C2 step (for ncu captures): python scripts/prof_c2.py [steps]"""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch, synth
import paper_1602_02740_b200 as tg
steps = int(sys.argv[1]) if len(sys.argv) > 1 else 1
u, v = synth.config_inputs(2)
u, v = torch.from_numpy(u).cuda(), torch.from_numpy(v).cuda()
for _ in range(steps):
    w = tg.toom_mul_batched(u, v, B=4, t4=32, t3=32)
torch.cuda.synchronize()
print("ok", w.shape)
