/*
 * mp_kernels.h — kernel-level entry points of libmpsolve.so, for unit tests of
 * individual steps of the hot path (not needed to solve a system).
 *
 * mp_kernel_schur_update: the trailing (Schur complement) update of the blocked
 * LU, PAPER.md P:139-142 / SGETRF: on a ROW-major binary32 matrix W
 * (device pointer, leading dimension ldw, the library's working-copy layout)
 *     W[r0+i][c0+j] -= sum_k W[r0+i][k0+k] * W[k0+k][c0+j],  i < M, j < N, k < K.
 * variant: MP_VARIANT_FFMA (CUDA-core FFMA) or MP_VARIANT_3XTF32 (tcgen05 tensor
 * cores, hi/lo TF32 split) or MP_VARIANT_TF32, in bits 0-7; bits 8-11: cluster size (1, 2
 * or 4) of the tcgen05 kernel — CTAs of a cluster take neighbouring tiles of a tile row and
 * share the L21 boxes by TMA multicast — 0 = the library's policy (MP_GEMM_CLUSTER, clusters
 * only for launches of several waves of tiles).  Runs on the library stream (mp_set_stream) and is
 * synchronous.  Returns MP_OK or MP_ERR_* (see mp_solve.h).
 *
 * mp_kernel_schur_update_f64: the same update on a row-major binary64 W — DGETRF's
 * trailing update of the binary64 path (mp_dgesv / the fallback, P:365-368 in binary64,
 * T3's reference solve P:393-394).  pipe: MP_F64_AUTO (the library's choice: DMMA tiles
 * when N, K and the row starts are even, else DFMA), MP_F64_DMMA (FP64 tensor pipe,
 * mma.sync m8n8k4; MP_ERR_UNSUPPORTED if the shape is not even), MP_F64_DFMA (CUDA-core
 * DFMA tile kernel).  Synchronous.
 */
#define MP_F64_AUTO 0
#define MP_F64_DMMA 1
#define MP_F64_DFMA 2
#ifndef MP_KERNELS_H
#define MP_KERNELS_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

int mp_kernel_schur_update(float *W, int64_t ldw, int64_t r0, int64_t c0, int64_t k0, int64_t M, int64_t N,
                           int64_t K, int variant);
int mp_kernel_schur_update_f64(double *W, int64_t ldw, int64_t r0, int64_t c0, int64_t k0, int64_t M, int64_t N,
                               int64_t K, int pipe);

#ifdef __cplusplus
}
#endif

#endif /* MP_KERNELS_H */
