"""Host logic of the 1D block-cyclic multi-GPU path with torch.distributed
(gloo, world size 2, CPU): column ownership, per-block seeded generation independent of P,
the distributed right-hand side (all-reduce of A_local x_local) and the id exchange.  These
are the same helpers bench.py --gpus N runs under NCCL."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as tmp

from paper_0808_2794_b200 import binding as mp
from paper_0808_2794_b200 import dist as pd


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, n, nb, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        cols = mp.local_columns(n, nb, world, rank)
        Al = pd.gen_local_A(n, nb, world, rank, seed=11, device="cpu")
        xt = pd.gen_xtrue(n, 2, seed=11, device="cpu")
        B = pd.distributed_rhs(Al, xt, cols)
        uid = pd.exchange_uid(rank, lambda: bytes(range(128)))
        # every rank's columns, gathered for the check on rank 0
        parts = [None] * world
        dist.all_gather_object(parts, (cols.tolist(), Al.numpy().copy()))
        q.put((rank, B.numpy().copy(), uid, parts))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("n,nb", [(300, 64), (257, 128)])
def test_block_cyclic_host_logic_gloo(n, nb):
    world = 2
    ctx = tmp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, n, nb, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = [q.get(timeout=300) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    res.sort(key=lambda t: t[0])
    # ownership: disjoint, complete, block j on rank j % P, counts as the C-ABI reports
    parts = res[0][3]
    allc = np.concatenate([np.asarray(c) for c, _ in parts])
    assert np.array_equal(np.sort(allc), np.arange(n))
    for r, (c, _) in enumerate(parts):
        assert all((ci // nb) % world == r for ci in c)
        assert len(c) == mp.mp_1dbc_local_cols(n, nb, world, r)
    # the assembled matrix equals the single-rank generation (independent of P)
    A = np.zeros((n, n))
    for c, a in parts:
        A[:, c] = a
    A1 = pd.gen_local_A(n, nb, 1, 0, seed=11, device="cpu").numpy()
    assert np.array_equal(A, A1)
    # distributed right-hand side = A x_true on every rank; identical ids
    xt = pd.gen_xtrue(n, 2, seed=11, device="cpu").numpy()
    for r in range(world):
        assert np.allclose(res[r][1], A @ xt, rtol=1e-12, atol=1e-10)
        assert res[r][2] == bytes(range(128))
    assert np.array_equal(res[0][1], res[1][1])
