"""C5 (BASELINE.json configs[4]) with the 31 top-level products sharded over
the GPUs of one node (paper_1602_02740_b200/dist.py; Eq. 2.5).

    python -m torch.distributed.run --nproc-per-node N --master-addr 127.0.0.1 \
        scripts/c5_sharded.py [--steps K] [--warmup W] [--n LIMBS]

Rank 0 evaluates, NCCL scatters the evaluated pairs, every rank multiplies
its share, NCCL gathers the products, rank 0 interpolates.  Prints one JSON
line on rank 0: ms per product (max over ranks, CUDA events) and a residue
check of the result (mod 8 seeded 61-bit primes) against the inputs.
"""
import argparse
import json
import os
import sys

import torch
import torch.distributed as dist

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import synth  # noqa: E402
from paper_1602_02740_b200 import dist as tgdist  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--steps", type=int, default=3)
    ap.add_argument("--warmup", type=int, default=1)
    ap.add_argument("--n", type=int, default=1 << 24)
    args = ap.parse_args()
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if world > 1:
        dist.init_process_group("nccl", device_id=dev)
    n = args.n
    u = v = None
    if rank == 0:
        seed = synth.seed_for(5)
        if n == 1 << 24:
            un, vn = synth.config_inputs(5)
        else:
            un = synth.uniform_limbs(seed, 0, 1, 0, n)[0]
            vn = synth.uniform_limbs(seed, 0, 1, 1, n)[0]
        u, v = torch.from_numpy(un).to(dev), torch.from_numpy(vn).to(dev)
    ops = tgdist.CudaOps(B=16)
    w = None
    for _ in range(args.warmup):
        w = tgdist.sharded_mul(u, v, n, ops, device=dev)
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(args.steps):
        w = tgdist.sharded_mul(u, v, n, ops, device=dev)
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / args.steps
    if world > 1:
        t = torch.tensor([ms], dtype=torch.float64, device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms = float(t.item())
    if rank == 0:
        import oracle   # residue check only (test infrastructure), after the timed region
        un, vn, wn = u.cpu().numpy(), v.cpu().numpy(), w.cpu().numpy()
        ok = all(oracle.residue(wn, p) == oracle.residue(un, p) * oracle.residue(vn, p) % p
                 for p in oracle.primes(synth.PRIME_SEED, 8))
        print(json.dumps({"workload": "C5 sharded top level (31-point Toom-16)", "n_limbs": n, "n_gpus": world,
                          "ms_per_product": ms, "steps": args.steps, "residues_ok": ok,
                          "shards": [hi - lo for lo, hi in tgdist.shard_bounds(31, world)[0]]}), flush=True)
    if world > 1:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
