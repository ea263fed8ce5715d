"""Kernel-level parity (`-m gpu`): the Schur update K5 (FFMA and tcgen05 3xTF32) through
the C-ABI test hook include/mp_kernels.h, against an fp64 reference of the same op."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def mp():
    torch = pytest.importorskip("torch")
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_0808_2794_b200 import build
    build.build()
    from paper_0808_2794_b200 import binding
    return binding


def run(mp, W0, r0, c0, k0, M, N, K, variant):
    import torch
    ldw = W0.shape[1]
    W = torch.from_numpy(W0.copy()).cuda()
    mp.mp_kernel_schur_update(W, r0, c0, k0, M, N, K, variant)
    torch.cuda.synchronize()
    assert W.stride(0) == ldw
    return W.cpu().numpy()


def reference(W0, r0, c0, k0, M, N, K):
    W = W0.astype(np.float64)
    R = W.copy()
    R[r0:r0 + M, c0:c0 + N] -= W[r0:r0 + M, k0:k0 + K] @ W[k0:k0 + K, c0:c0 + N]
    return R


SHAPES = [(64, 64, 0, 256, 128, 64), (300, 200, 7, 512, 333, 32), (1000, 700, 16, 1400, 1200, 256),
          (256, 128, 0, 300, 400, 100), (513, 129, 40, 700, 700, 200), (2048, 2048, 256, 2304, 2304, 256)]


@pytest.mark.parametrize("variant", [0, 1])
@pytest.mark.parametrize("shape", SHAPES)
def test_schur_update_exact_integers(mp, variant, shape):
    """Small integers: every product and partial sum is exact in fp32 (and tf32 hi, lo = 0)."""
    M, N, k0, rows, cols, K = shape
    rng = np.random.default_rng(M + N + K)
    ldw = ((cols + 63) // 64) * 64
    W0 = rng.integers(-8, 9, size=(rows, ldw)).astype(np.float32)
    r0, c0 = k0 + K, k0 + K
    M, N = min(M, rows - r0), min(N, cols - c0)
    got = run(mp, W0, r0, c0, k0, M, N, K, variant)
    ref = reference(W0, r0, c0, k0, M, N, K)
    assert np.array_equal(got.astype(np.float64), ref)


@pytest.mark.parametrize("variant", [0, 1])
def test_schur_update_gaussian_accuracy(mp, variant):
    rng = np.random.default_rng(5)
    rows = cols = 1536
    W0 = rng.standard_normal((rows, cols)).astype(np.float32)
    k0, K = 256, 256
    r0 = c0 = k0 + K
    M, N = rows - r0, cols - c0
    got = run(mp, W0, r0, c0, k0, M, N, K, variant)
    ref = reference(W0, r0, c0, k0, M, N, K)
    scale = np.abs(W0[r0:, k0:k0 + K]).astype(np.float64) @ np.abs(W0[k0:k0 + K, c0:]).astype(np.float64)
    err = np.abs(got[r0:, c0:] - ref[r0:, c0:]) / (scale + np.abs(ref[r0:, c0:]))
    # fp32 accumulation over K terms: ~K * 2^-24; 3xTF32 adds the dropped lo*lo term and tf32 rounding of lo
    assert err.max() <= K * 2.0 ** -24 * 4, err.max()
    # untouched regions stay bitwise
    assert np.array_equal(got[:r0], W0[:r0]) and np.array_equal(got[:, :c0], W0[:, :c0])


CLUSTER_SHAPES = [(300, 200, 7, 512, 333, 32), (1000, 700, 16, 1400, 1200, 256), (513, 129, 40, 700, 700, 200),
                  (256, 1300, 0, 600, 1700, 256), (2048, 2048, 256, 2304, 2304, 256)]


@pytest.mark.parametrize("cluster", [1, 2, 4, 8])
@pytest.mark.parametrize("shape", CLUSTER_SHAPES)
def test_schur_update_clusters_exact_and_bitwise(mp, cluster, shape):
    """The tcgen05 update with its L boxes multicast over clusters of 2 / 4 CTAs (variant bits 8-11):
    exact on small integers (odd tile counts: a cluster's surplus CTA stores nothing) and, on
    Gaussian data, bitwise equal to the single-CTA kernel (same MMA order per tile).  cluster = 8
    selects the CTA-pair kernel (tcgen05 cta_group::2: one 256 x 256 instruction tile per pair)."""
    M, N, k0, rows, cols, K = shape
    rng = np.random.default_rng(M + N + K + cluster)
    ldw = ((cols + 63) // 64) * 64
    W0 = rng.integers(-8, 9, size=(rows, ldw)).astype(np.float32)
    r0, c0 = k0 + K, k0 + K
    M, N = min(M, rows - r0), min(N, cols - c0)
    got = run(mp, W0, r0, c0, k0, M, N, K, 1 | (cluster << 8))
    assert np.array_equal(got.astype(np.float64), reference(W0, r0, c0, k0, M, N, K))
    G0 = rng.standard_normal((rows, ldw)).astype(np.float32)
    one = run(mp, G0, r0, c0, k0, M, N, K, 1 | (1 << 8))
    got = run(mp, G0, r0, c0, k0, M, N, K, 1 | (cluster << 8))
    assert np.array_equal(got, one)
    got1 = run(mp, G0, r0, c0, k0, M, N, K, 2 | (cluster << 8))     # 1xTF32 (hi boxes only)
    assert np.array_equal(got1, run(mp, G0, r0, c0, k0, M, N, K, 2 | (1 << 8)))


# --------------------------------------------------------------------------- binary64 update (FP64 path)
def run64(mp, W0, r0, c0, k0, M, N, K, pipe):
    import torch
    W = torch.from_numpy(W0.copy()).cuda()
    mp.mp_kernel_schur_update_f64(W, r0, c0, k0, M, N, K, pipe)
    torch.cuda.synchronize()
    return W.cpu().numpy()


SHAPES64 = [(64, 64, 0, 256, 128, 64), (300, 200, 8, 512, 334, 32), (1000, 700, 16, 1400, 1200, 256),
            (513, 130, 40, 700, 700, 200), (2048, 2048, 256, 2304, 2304, 256), (333, 257, 3, 600, 600, 61)]


@pytest.mark.parametrize("pipe", [0, 1, 2])
@pytest.mark.parametrize("shape", SHAPES64)
def test_schur_update_f64_exact_integers(mp, pipe, shape):
    """Integers: every product and partial sum is exact in binary64, so any order gives the same bits.
    pipe 1 (DMMA) needs even N, K and row starts: the odd last shape must be refused; pipe 0
    (the library's routing) falls back to the DFMA kernel there."""
    M, N, k0, rows, cols, K = shape
    rng = np.random.default_rng(M + N + K + 1)
    ldw = ((cols + 63) // 64) * 64
    W0 = rng.integers(-64, 65, size=(rows, ldw)).astype(np.float64)
    r0, c0 = k0 + K, k0 + K
    M, N = min(M, rows - r0), min(N, cols - c0)
    if pipe == 1 and (N % 2 or K % 2 or k0 % 2 or c0 % 2):
        with pytest.raises(mp.MpError):
            run64(mp, W0, r0, c0, k0, M, N, K, pipe)
        return
    got = run64(mp, W0, r0, c0, k0, M, N, K, pipe)
    ref = reference(W0, r0, c0, k0, M, N, K)
    assert np.array_equal(got, ref)


@pytest.mark.parametrize("pipe", [1, 2])
def test_schur_update_f64_gaussian_accuracy(mp, pipe):
    rng = np.random.default_rng(6)
    rows = cols = 1536
    W0 = rng.standard_normal((rows, cols))
    k0, K = 256, 256
    r0 = c0 = k0 + K
    M, N = rows - r0, cols - c0
    got = run64(mp, W0, r0, c0, k0, M, N, K, pipe)
    exact = W0[r0:, c0:].astype(np.longdouble) - W0[r0:, k0:k0 + K].astype(np.longdouble) @ W0[k0:k0 + K, c0:].astype(np.longdouble)
    scale = np.abs(W0[r0:, k0:k0 + K]) @ np.abs(W0[k0:k0 + K, c0:]) + np.abs(W0[r0:, c0:])
    err = np.abs(got[r0:, c0:] - np.asarray(exact, np.float64)) / scale
    assert err.max() <= (K + 1) * 2.0 ** -53, err.max()         # binary64 accumulation bound
    assert np.array_equal(got[:r0], W0[:r0]) and np.array_equal(got[:, :c0], W0[:, :c0])
