"""Host-side helpers of the 1D block-cyclic multi-GPU path: seeded generation of
each rank's column blocks, the distributed right-hand side, and the NCCL unique-id exchange.
No method arithmetic (the solver runs in libmpsolve.so); torch.distributed is plumbing only.

Column block j (nb columns) is owned by rank j % P.  Each block is generated from its own
seed (seed, j), so the assembled matrix does not depend on P: a rank generates only its blocks.
"""
from __future__ import annotations

import numpy as np

from .binding import local_columns


def _gen(device: str, seed: int):
    import torch
    g = torch.Generator(device=device)
    g.manual_seed(int(seed))
    return g


def block_seed(seed: int, j: int) -> int:
    return (int(seed) * 1_000_003 + 7919 * j + 1) % (2 ** 63 - 1)


def gen_block(n: int, nb: int, j: int, seed: int, device: str = "cuda"):
    """Column block j of A (n x min(nb, n - j nb)), i.i.d. N(0,1), column-major (stride (1, n))."""
    import torch
    w = min(nb, n - j * nb)
    return torch.randn((w, n), dtype=torch.float64, device=device, generator=_gen(device, block_seed(seed, j))).t()


def gen_local_A(n: int, nb: int, nranks: int, rank: int, seed: int, device: str = "cuda"):
    """This rank's columns of A (n x local_cols, column-major), blocks in increasing global order."""
    import torch
    nblk = -(-n // nb)
    ncols = len(local_columns(n, nb, nranks, rank))
    out = torch.empty((ncols, n), dtype=torch.float64, device=device).t()
    c = 0
    for j in range(rank, nblk, nranks):
        blk = gen_block(n, nb, j, seed, device)
        out[:, c:c + blk.shape[1]] = blk
        c += blk.shape[1]
    return out


def gen_xtrue(n: int, nrhs: int, seed: int, device: str = "cuda"):
    """x_true i.i.d. U[-1, 1] (n x nrhs, column-major)."""
    import torch
    g = _gen(device, block_seed(seed, 10 ** 7))
    return (torch.rand((nrhs, n), dtype=torch.float64, device=device, generator=g) * 2 - 1).t()


def distributed_rhs(A_local, x_true, cols, group=None):
    """B = A x_true = sum over ranks of A_local x_true[cols] (all-reduce), replicated, column-major."""
    import torch
    import torch.distributed as dist
    idx = torch.as_tensor(np.asarray(cols, dtype=np.int64), device=x_true.device)
    part = A_local @ x_true.index_select(0, idx) if len(cols) else torch.zeros_like(x_true)
    part = part.t().contiguous()                       # (nrhs, n) row-major = column-major (n, nrhs)
    if dist.is_initialized() and dist.get_world_size() > 1:
        dist.all_reduce(part, op=dist.ReduceOp.SUM, group=group)
    return part.t()


def exchange_uid(rank: int, make_uid):
    """Rank 0 creates the communicator id (make_uid() -> bytes); every rank receives it."""
    import torch.distributed as dist
    obj = [make_uid() if rank == 0 else None]
    if dist.is_initialized() and dist.get_world_size() > 1:
        dist.broadcast_object_list(obj, src=0)
    return obj[0]
