"""Multi-process (world_size 2 and 3, gloo on CPU) test of the sharded top
level of C5 (paper_1602_02740_b200/dist.py): u and v are broadcast, every
rank evaluates and multiplies its own points, the products are gathered and
interpolated on rank 0 (Eq. 2.5).

The compute steps are exact-integer stand-ins written here from the
definitions (test infrastructure): homogeneous evaluation
sum_j u_j p^j q^(n-j) (Eq. 1.1-1.2), exact signed products, and
interpolation by solving the homogeneous Vandermonde system with Fractions.
What is under test is the partition and the exchange (shapes, padding, order,
which rank owns which point), not the kernels (tests/test_gpu_parity.py).
"""
import os
import socket
from fractions import Fraction

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import synth
from paper_1602_02740_b200 import dist as tgdist

# the 31-point set of configs[4] (SURVEY §8(c) reading 5), written out
POINTS = [(0, 1), (1, 0), (1, 1), (-1, 1), (2, 1), (-2, 1), (1, 2), (-1, 2), (3, 1), (-3, 1), (1, 3), (-1, 3),
          (3, 2), (-3, 2), (2, 3), (-2, 3), (4, 1), (-4, 1), (1, 4), (-1, 4), (4, 3), (-4, 3), (3, 4), (-3, 4),
          (5, 1), (-5, 1), (1, 5), (-1, 5), (5, 2), (-5, 2), (2, 5)]
B = 16


def to_limbs(x, w):
    x %= 1 << (32 * w)
    return np.array([(x >> (32 * i)) & 0xFFFFFFFF for i in range(w)], dtype=np.uint32)


def from_limbs(a, signed=True):
    x = synth.to_int(a)
    if signed and len(a) and (int(a[-1]) >> 31):
        x -= 1 << (32 * len(a))
    return x


class IntOps:
    """Exact-integer stand-ins for the three stage exports."""

    def widths(self, n):
        b = -(-n // B)
        return len(POINTS), b + 2

    def blocks(self, a, n):
        b = -(-n // B)
        x = synth.to_int(a.numpy())
        return [(x >> (32 * b * j)) & ((1 << (32 * b)) - 1) for j in range(B)]

    def eval_points(self, a):
        n = a.numel()
        _, e = self.widths(n)
        blk = self.blocks(a, n)
        rows = [to_limbs(sum(c * p**j * q ** (B - 1 - j) for j, c in enumerate(blk)), e) for p, q in POINTS]
        return torch.from_numpy(np.stack(rows))

    def eval_range(self, a, k0, k1):
        return self.eval_points(a)[k0:k1].contiguous()

    def mul(self, U, V):
        e = U.shape[1]
        rows = [to_limbs(from_limbs(U[i].numpy()) * from_limbs(V[i].numpy()), 2 * e) for i in range(U.shape[0])]
        return torch.from_numpy(np.stack(rows)) if rows else torch.zeros((0, 2 * e), dtype=torch.uint32)

    def interp(self, Y, n):
        d = 2 * B - 2
        ys = [Fraction(from_limbs(Y[k].numpy())) for k in range(Y.shape[0])]
        A = [[Fraction(p**j * q ** (d - j)) for j in range(d + 1)] for p, q in POINTS]
        # Gauss-Jordan on [A | y]
        M = [row + [y] for row, y in zip(A, ys)]
        for c in range(d + 1):
            piv = next(r for r in range(c, d + 1) if M[r][c] != 0)
            M[c], M[piv] = M[piv], M[c]
            inv = 1 / M[c][c]
            M[c] = [x * inv for x in M[c]]
            for r in range(d + 1):
                if r != c and M[r][c] != 0:
                    f = M[r][c]
                    M[r] = [x - f * y for x, y in zip(M[r], M[c])]
        w = [M[j][d + 1] for j in range(d + 1)]
        assert all(x.denominator == 1 for x in w)
        b = -(-n // B)
        tot = sum(int(x) << (32 * b * j) for j, x in enumerate(w))
        return torch.from_numpy(to_limbs(tot, 2 * n))


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, n, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        seed = synth.seed_for(5)
        u = torch.from_numpy(synth.uniform_limbs(seed, 3, 1, 0, n)[0]) if rank == 0 else None
        v = torch.from_numpy(synth.uniform_limbs(seed, 3, 1, 1, n)[0]) if rank == 0 else None
        w = tgdist.sharded_mul(u, v, n, IntOps())
        if rank == 0:
            q.put(synth.to_int(w.numpy()) == synth.to_int(u.numpy()) * synth.to_int(v.numpy()))
        else:
            q.put(w is None)
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
def test_sharded_top_level_gloo(world):
    n = 64
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    ps = [ctx.Process(target=_worker, args=(r, world, port, n, q)) for r in range(world)]
    for p in ps:
        p.start()
    res = [q.get(timeout=300) for _ in ps]
    for p in ps:
        p.join(timeout=60)
    assert all(res) and len(res) == world


def test_shard_bounds():
    b, m = tgdist.shard_bounds(31, 8)
    assert m == 4 and [hi - lo for lo, hi in b] == [4, 4, 4, 4, 4, 4, 4, 3]
    b, m = tgdist.shard_bounds(31, 2)
    assert [hi - lo for lo, hi in b] == [16, 15]
    b, m = tgdist.shard_bounds(31, 1)
    assert b == [(0, 31)]


def test_single_rank_path_int_ops():
    seed = synth.seed_for(5)
    n = 48
    u = torch.from_numpy(synth.uniform_limbs(seed, 4, 1, 0, n)[0])
    v = torch.from_numpy(synth.uniform_limbs(seed, 4, 1, 1, n)[0])
    w = tgdist.sharded_mul(u, v, n, IntOps())
    assert synth.to_int(w.numpy()) == synth.to_int(u.numpy()) * synth.to_int(v.numpy())


# ---------------------------------------------------------------- C2 slices
# bench.py splits the ONE C2 batch into contiguous slices of 65536/P products
# (strong scaling); each rank generates its own slice from
# the counter-based stream.  Check with gloo ranks that the slices partition
# the batch and that the per-rank inputs are exactly the full batch's rows.

def _c2_worker(rank, world, port, total, q):
    import sys
    sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
    import bench
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        lo, hi = bench.c2_slice(rank, world, total)
        u, v = bench.c2_inputs(lo, hi, 16)
        # exact products of this slice (Python integers; the compute is not under test)
        w = np.stack([to_limbs(synth.to_int(a) * synth.to_int(b), 32) for a, b in zip(u, v)])
        m = -(-total // world)
        pad = np.zeros((m, 32), np.uint32)
        pad[: hi - lo] = w
        gl = [torch.zeros((m, 32), dtype=torch.int32) for _ in range(world)]
        cnt = [torch.zeros(1, dtype=torch.int64) for _ in range(world)]
        dist.all_gather(gl, torch.from_numpy(pad.view(np.int32)))
        dist.all_gather(cnt, torch.tensor([hi - lo]))
        if rank == 0:
            rows = np.concatenate([g.numpy().view(np.uint32)[: int(c)] for g, c in zip(gl, cnt)])
            uf, vf = bench.c2_inputs(0, total, 16)
            want = np.stack([to_limbs(synth.to_int(a) * synth.to_int(b), 32) for a, b in zip(uf, vf)])
            q.put(rows.shape[0] == total and np.array_equal(rows, want))
        else:
            q.put(True)
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
def test_c2_strong_scaling_slices_gloo(world):
    total = 101
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    ps = [ctx.Process(target=_c2_worker, args=(r, world, port, total, q)) for r in range(world)]
    for p in ps:
        p.start()
    res = [q.get(timeout=300) for _ in ps]
    for p in ps:
        p.join(timeout=60)
    assert all(res) and len(res) == world


def test_c2_slices_partition_the_batch():
    import sys
    sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
    import bench
    for world in (1, 2, 3, 4, 8):
        s = [bench.c2_slice(r, world) for r in range(world)]
        assert s[0][0] == 0 and s[-1][1] == 65536
        assert all(s[i][1] == s[i + 1][0] for i in range(world - 1))
        assert max(h - l for l, h in s) - min(h - l for l, h in s) <= 1
