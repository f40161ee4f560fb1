"""SURVEY §8(f)2 measurement: the base case on the int8 tensor cores
(toom_base_interleaved_tc) against the IMAD.WIDE.U32 path
(toom_base_interleaved) on the C2 and C4 base-case batches:
python scripts/time_tc_base.py [reps]"""
import json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_1602_02740_b200 as tg
reps = int(sys.argv[1]) if len(sys.argv) > 1 else 5
for E, count, what in [(18, 65536 * 49, "C2 base batch (49 products of 18 limbs per C2 product)"),
                       (23, 823543 * 5, "C4 base batch (5 products of 23 limbs per fused T3 instance)")]:
    g = torch.Generator(device="cuda").manual_seed(E)
    u = torch.randint(0, 2**31, (E, count), dtype=torch.int64, device="cuda", generator=g).to(torch.uint32)
    v = torch.randint(0, 2**31, (E, count), dtype=torch.int64, device="cuda", generator=g).to(torch.uint32)
    res = {"E": E, "count": count, "workload": what}
    outs = {}
    for name, fn in (("imad", tg.base_interleaved), ("tcgen05_i8", tg.base_interleaved_tc)):
        outs[name] = fn(u, v)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(reps):
            fn(u, v)
        e1.record(); torch.cuda.synchronize()
        ms = e0.elapsed_time(e1) / reps
        res[name] = {"ms": ms, "products_per_s": count / (ms * 1e-3), "limb_products_per_s": count * E * E / (ms * 1e-3)}
    res["equal"] = bool(torch.equal(outs["imad"], outs["tcgen05_i8"]))
    res["tc_over_imad_time"] = res["tcgen05_i8"]["ms"] / res["imad"]["ms"]
    print(json.dumps(res), flush=True)
