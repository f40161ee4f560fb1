"""Sharded top level of one large product (BASELINE.json configs[4], C5;
SURVEY.md §8(e), call stack (4)).

The paper puts the 2B-1 top-level products of one multiplication on P
processors (Eq. 2.5: T = (1/P) N^alpha).  Here the processors
are GPUs, one process per GPU:

  1. broadcast: u and v reach every rank               (NCCL over NVLink)
  2. rank r evaluates u and v at its own points
     k in [r m, (r+1) m), m = ceil((2B-1)/P)           (toom_eval_points_range)
  3. every rank multiplies its pairs (recursive Toom-4/3 on the GPU,
     toom_mul_signed_batched)
  4. gather: the products y_k return to rank 0         (NCCL)
  5. rank 0 interpolates and recomposes w              (toom_interp_recompose)
Rank 0's serial part is the interpolation alone: the evaluation is split P
ways (the broadcast moves 2n limbs, the scatter of evaluated pairs moved
(2B-1)(n/B) x 2).

The compute steps are the C-ABI calls of libtoomgpu; this module only moves
tensors between ranks.  `ops` can be replaced (tests run the exchange logic
on CPU with the gloo backend and exact-integer stand-ins).
"""
from __future__ import annotations

import math

import torch
import torch.distributed as dist


class CudaOps:
    """The product path: libtoomgpu's long-path stage exports."""

    def __init__(self, B: int = 16, t4: int = 256, t3: int = 64):
        from . import eval_points, eval_points_range, interp_recompose, lib, mul_signed_batched
        self._ev, self._evr, self._ir, self._mul = eval_points, eval_points_range, interp_recompose, mul_signed_batched
        self.B, self.t4, self.t3 = B, t4, t3
        self.lib = lib()

    def widths(self, n: int):
        return self.lib.toom_npoints(self.B), self.lib.toom_eval_width(n, self.B)

    def eval_points(self, a: torch.Tensor) -> torch.Tensor:          # [n] -> [npts][e]
        return self._ev(a.view(1, -1), self.B)[:, 0, :].contiguous()

    def eval_range(self, a: torch.Tensor, k0: int, k1: int) -> torch.Tensor:   # [n] -> [k1-k0][e]
        return self._evr(a.view(1, -1), self.B, k0, k1)[:, 0, :].contiguous()

    def mul(self, U: torch.Tensor, V: torch.Tensor) -> torch.Tensor:   # [m][e] x2 -> [m][2e]
        if U.shape[0] == 0:
            return torch.empty((0, 2 * U.shape[1]), dtype=U.dtype, device=U.device)
        return self._mul(U, V, B=4, t4=self.t4, t3=self.t3)

    def interp(self, Y: torch.Tensor, n: int) -> torch.Tensor:        # [npts][2e] -> [2n]
        return self._ir(Y.view(Y.shape[0], 1, Y.shape[1]), n, self.B)[0]


def shard_bounds(npts: int, world: int):
    """Contiguous point ranges, ceil(npts/world) per rank (the last ones may
    be short or empty): 31 points on 8 ranks -> 4,4,4,4,4,4,4,3."""
    m = math.ceil(npts / world)
    return [(min(r * m, npts), min((r + 1) * m, npts)) for r in range(world)], m


def sharded_mul(u, v, n: int, ops, group=None, device=None):
    """w = u*v with the top-level products sharded over the ranks of `group`.
    u, v: 1-D [n] uint32 tensors on rank 0 (ignored elsewhere).  Returns the
    2n-limb product on rank 0, None on the other ranks."""
    rank = dist.get_rank(group) if dist.is_initialized() else 0
    world = dist.get_world_size(group) if dist.is_initialized() else 1
    npts, e = ops.widths(n)
    bounds, m = shard_bounds(npts, world)
    dev = device if device is not None else (u.device if rank == 0 else torch.device("cpu"))
    if world == 1:
        return ops.interp(ops.mul(ops.eval_points(u), ops.eval_points(v)), n)

    # 1: broadcast u, v (limbs travel as int32: same bits); 2: evaluate this
    # rank's points
    i32 = torch.int32
    if rank == 0:
        ub, vb = u.contiguous().view(i32), v.contiguous().view(i32)
    else:
        ub = torch.empty(n, dtype=i32, device=dev)
        vb = torch.empty(n, dtype=i32, device=dev)
    dist.broadcast(ub, src=0, group=group)
    dist.broadcast(vb, src=0, group=group)
    lo, hi = bounds[rank]
    k = hi - lo
    # 3: this rank's products (real rows only; the gather pads to m rows)
    U = ops.eval_range(ub.view(torch.uint32), lo, hi)
    V = ops.eval_range(vb.view(torch.uint32), lo, hi)
    Y = ops.mul(U, V)
    Ysend = torch.zeros((m, 2 * e), dtype=i32, device=dev)
    if k:
        Ysend[:k] = Y.view(i32)
    # 4: gather the products on rank 0
    if rank == 0:
        gl = [torch.empty((m, 2 * e), dtype=i32, device=dev) for _ in range(world)]
        dist.gather(Ysend, gl, dst=0, group=group)
        Yall = torch.cat(gl)[:npts].contiguous().view(torch.uint32)
        # 5: interpolation + recomposition
        return ops.interp(Yall, n)
    dist.gather(Ysend, None, dst=0, group=group)
    return None
