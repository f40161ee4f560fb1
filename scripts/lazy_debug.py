import os, sys, json
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_1602_02740_b200 as tg
rng = np.random.default_rng(1)
for (B, n, batch) in [(4, 4100, 9), (4, 4100, 1), (4, 3001, 1), (4, 1 << 13, 1), (4, 1 << 14, 3), (16, 1 << 13, 1), (4, 20000, 2)]:
    u = rng.integers(0, 2**32, (batch, n), dtype=np.uint64).astype(np.uint32)
    v = rng.integers(0, 2**32, (batch, n), dtype=np.uint64).astype(np.uint32)
    w = tg.toom_mul_batched(torch.from_numpy(u).cuda(), torch.from_numpy(v).cuda(), B=B).cpu().numpy()
    ok = [int.from_bytes(w[i].tobytes(), 'little') == int.from_bytes(u[i].tobytes(), 'little') * int.from_bytes(v[i].tobytes(), 'little') for i in range(batch)]
    d = tg.plan_describe(n, batch, B=B)
    print(B, n, batch, ok, [(l['count'], l['n'], l['lazy']) for l in d['levels']], flush=True)
