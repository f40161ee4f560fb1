"""Small invocations of every kernel family for compute-sanitizer (memcheck /
racecheck / synccheck): python scripts/sanitize_small.py"""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import synth, oracle
import paper_1602_02740_b200 as tg
ok = True
def chk(name, got, want):
    global ok
    good = np.array_equal(got, want)
    ok &= good
    print(name, "ok" if good else "MISMATCH", flush=True)
d = lambda a: torch.from_numpy(np.ascontiguousarray(a)).cuda()
u, v = synth.config_inputs(1, batch=10, first=250)
chk("C1 fused top", tg.toom_mul_batched(d(u), d(v), B=3, t4=10**9, t3=10**9).cpu().numpy(), oracle.schoolbook_batched(u, v))
u, v = synth.config_inputs(2, batch=70)
chk("C2 eval/fused/interp", tg.toom_mul_batched(d(u), d(v), B=4, t4=32, t3=32).cpu().numpy(), oracle.schoolbook_batched(u, v))
u, v = synth.config_inputs(3, batch=6, first=1020)
chk("C3 P8 rows + recompose", tg.toom_mul_batched(d(u), d(v), B=8).cpu().numpy(), oracle.schoolbook_batched(u, v))
rng = np.random.default_rng(1)
a = rng.integers(0, 2**32, 5000, dtype=np.uint64).astype(np.uint32)
b = rng.integers(0, 2**32, 5000, dtype=np.uint64).astype(np.uint32)
chk("long path T4", tg.toom_mul(d(a), d(b), B=4).cpu().numpy(), oracle.schoolbook(a, b))
chk("long path T16", tg.toom_mul(d(a), d(b), B=16).cpu().numpy(), oracle.schoolbook(a, b))
print("ALL OK" if ok else "FAILURES")
