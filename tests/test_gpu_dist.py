"""1D block-cyclic multi-GPU path, exercised on ONE GPU with the loopback
communicator: P emulated ranks are P host threads of this process, each with its own stream;
collectives meet at a host barrier (no kernel waits on another rank's kernel).  The same
solver code runs over NCCL with one process per GPU (bench.py --gpus N)."""
import threading

import numpy as np
import pytest

import oracle as orc_mod
from paper_0808_2794_b200 import inputs

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def mp():
    import torch
    assert torch.cuda.is_available()
    from paper_0808_2794_b200 import binding
    return binding


def run_dist(mp, A, B, nranks, nb, fp64=False, opts=None):
    import torch
    n = A.shape[0]
    comms = mp.mp_comm_init_loopback(nranks)
    out = [None] * nranks
    err = [None] * nranks

    def worker(r):
        try:
            torch.cuda.set_device(0)
            st = torch.cuda.Stream()
            with torch.cuda.stream(st):
                cols = mp.local_columns(n, nb, nranks, r)
                Al = mp.colmajor_cuda(A[:, cols]) if len(cols) else torch.zeros((n, 0), dtype=torch.float64, device="cuda")
                dB = mp.colmajor_cuda(B)
                if fp64:
                    X, info = mp.mp_dgesv_1dbc(comms[r], n, nb, Al, dB)
                    it = None
                else:
                    X, it, info, _ = mp.mp_dsgesv_1dbc_ex(comms[r], n, nb, Al, dB, opts=opts)
                st.synchronize()
                out[r] = (X.cpu().numpy().copy(order="F"), it, info)
        except BaseException as e:  # noqa: BLE001
            err[r] = e

    ts = [threading.Thread(target=worker, args=(r,)) for r in range(nranks)]
    for t in ts:
        t.start()
    for t in ts:
        t.join(timeout=600)
    for c in comms:
        mp.mp_comm_destroy(c)
    for e in err:
        if e is not None:
            raise e
    return out


def certificate_ok(A, X, B):
    n = A.shape[0]
    R = np.asarray(B, np.longdouble) - np.asarray(A, np.longdouble) @ np.asarray(X, np.longdouble)
    cte = np.linalg.norm(A) * 2.0 ** -53 * np.sqrt(n)
    return all(np.linalg.norm(np.asarray(R[:, c], float)) < 1.05 * np.linalg.norm(X[:, c]) * cte
               for c in range(X.shape[1]))


def test_local_cols_match_python(mp):
    for n, nb, P in [(1000, 256, 3), (4096, 128, 4), (300, 64, 8), (100, 256, 2)]:
        tot = 0
        for r in range(P):
            assert mp.mp_1dbc_local_cols(n, nb, P, r) == len(mp.local_columns(n, nb, P, r))
            tot += len(mp.local_columns(n, nb, P, r))
        assert tot == n


@pytest.mark.parametrize("nranks,n,nb", [(1, 700, 64), (2, 1000, 128), (3, 1100, 128), (4, 1500, 256)])
def test_dist_exact_lu_bitwise(mp, nranks, n, nb):
    A, B, X, *_ = inputs.exact_lu(n, nrhs=2, seed=n + nranks)
    for Xg, it, info in run_dist(mp, A, B, nranks, nb):
        assert (it, info) == (0, 0)
        assert np.array_equal(Xg, X)


@pytest.mark.parametrize("nranks,n,nrhs,nb,seed", [(2, 1024, 1, 128, 1), (3, 1500, 3, 128, 2), (4, 2300, 1, 256, 3)])
def test_dist_criterion_parity(mp, nranks, n, nrhs, nb, seed):
    A, B, Xt = inputs.gaussian(n, nrhs=nrhs, seed=seed)
    ro = orc_mod.dsgesv(A, B)
    res = run_dist(mp, A, B, nranks, nb)
    X0 = res[0][0]
    for Xg, it, info in res:
        assert info == 0 and ro.info == 0
        assert it >= 0 and abs(it - ro.iters) <= 1, (it, ro.iters)
        assert np.array_equal(Xg, X0)                  # every rank holds the same solution
    assert certificate_ok(A, X0, B)


def test_dist_fallback_and_dgesv(mp):
    n = 900
    A, B, X = inputs.conditioned(n, 1e10, seed=4)
    res = run_dist(mp, A, B, 2, 128)
    for Xg, it, info in res:
        assert it == -31 and info == 0
    ref = np.linalg.solve(A, B)
    kappa = 1e10
    assert np.abs(res[0][0] - ref).max() / np.abs(ref).max() < 1e-16 * kappa * n
    res64 = run_dist(mp, A, B, 3, 128, fp64=True)
    for Xg, _, info in res64:
        assert info == 0
        assert np.abs(Xg - ref).max() / np.abs(ref).max() < 1e-16 * kappa * n


def test_dist_ffma_variant(mp):
    A, B, Xt = inputs.gaussian(1200, nrhs=1, seed=7)
    ro = orc_mod.dsgesv(A, B)
    res = run_dist(mp, A, B, 2, 128, opts=mp.make_opts(variant=mp.MP_VARIANT_FFMA))
    for Xg, it, info in res:
        assert info == 0 and abs(it - ro.iters) <= 1
    assert certificate_ok(A, res[0][0], B)


def test_nccl_p1_communicator(mp):
    """The NCCL data plane on hardware: a real NCCL communicator of one rank (the driver's boxes
    have one GPU) runs mp_dsgesv_1dbc / mp_dgesv_1dbc, so NcclComm::bcast / allreduce / allgather
    execute through libnccl (a P = 1 broadcast / all-reduce / all-gather is still a real NCCL
    kernel on the stream).  Results against the oracle, and bitwise equal to the loopback P = 1
    run of the same algorithm."""
    import torch
    n, nb = 1100, 128
    A, B, Xt = inputs.gaussian(n, nrhs=2, seed=17)
    ro = orc_mod.dsgesv(A, B)
    uid = mp.mp_get_unique_id()
    comm = mp.mp_comm_init(1, 0, uid)
    try:
        dA, dB = mp.colmajor_cuda(A), mp.colmajor_cuda(B)
        X, it, info, rep = mp.mp_dsgesv_1dbc_ex(comm, n, nb, dA, dB)
        torch.cuda.synchronize()
        Xn = X.cpu().numpy()
        X64, info64 = mp.mp_dgesv_1dbc(comm, n, nb, dA, dB)
        torch.cuda.synchronize()
        X64 = X64.cpu().numpy()
    finally:
        mp.mp_comm_destroy(comm)
    assert info == ro.info == 0 and abs(it - ro.iters) <= 1, (it, ro.iters)
    assert certificate_ok(A, Xn, B)
    Xl, itl, infol = run_dist(mp, A, B, 1, nb)[0]
    assert (itl, infol) == (it, info) and np.array_equal(Xl, Xn)
    Xo, infoo = orc_mod.dgesv(A, B)
    kappa = np.linalg.cond(A)
    assert info64 == infoo == 0
    assert np.abs(X64 - Xo).max() / np.abs(Xo).max() <= 8 * n * kappa * 2.0 ** -53


@pytest.mark.parametrize("nranks,n,nrhs,nb", [(2, 900, 2, 128), (3, 1100, 7, 128), (4, 1000, 16, 256)])
def test_dist_split_rhs_solves(mp, nranks, n, nrhs, nb):
    """nrhs >= P: each rank solves its own right-hand-side columns and the solution is all-gathered
    (the refinement's solve work scales with P).  Same verdicts as the oracle, every rank holds the
    same X."""
    A, B, Xt = inputs.gaussian(n, nrhs=nrhs, seed=n + nranks)
    ro = orc_mod.dsgesv(A, B)
    res = run_dist(mp, A, B, nranks, nb)
    X0 = res[0][0]
    for Xg, it, info in res:
        assert info == 0 and ro.info == 0 and abs(it - ro.iters) <= 1, (it, ro.iters)
        assert np.array_equal(Xg, X0)
    assert certificate_ok(A, X0, B)
