"""Run the integer-MAD peak probes once (for ncu: python scripts/probe_run.py)."""
import os, sys, json
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_1602_02740_b200 as tg
torch.cuda.set_device(0)
r1, m1 = tg.probe_limb_products()
r2, m2 = tg.probe_carry_chain()
print(json.dumps({"imad_wide_lp_per_s": r1, "ms": m1, "carry_chain_lp_per_s": r2, "ms2": m2}))
