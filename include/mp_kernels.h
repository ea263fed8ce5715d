/*
 * mp_kernels.h — kernel-level entry points of libmpsolve.so, for unit tests of
 * individual steps of the hot path (not needed to solve a system).
 *
 * mp_kernel_schur_update: the trailing (Schur complement) update of the blocked
 * LU, PAPER.md P:139-142 / SGETRF: on a ROW-major binary32 matrix W
 * (device pointer, leading dimension ldw, the library's working-copy layout)
 *     W[r0+i][c0+j] -= sum_k W[r0+i][k0+k] * W[k0+k][c0+j],  i < M, j < N, k < K.
 * variant: MP_VARIANT_FFMA (CUDA-core FFMA) or MP_VARIANT_3XTF32 (tcgen05 tensor
 * cores, hi/lo TF32 split).  Runs on the library stream (mp_set_stream) and is
 * synchronous.  Returns MP_OK or MP_ERR_* (see mp_solve.h).
 */
#ifndef MP_KERNELS_H
#define MP_KERNELS_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

int mp_kernel_schur_update(float *W, int64_t ldw, int64_t r0, int64_t c0, int64_t k0, int64_t M, int64_t N,
                           int64_t K, int variant);

#ifdef __cplusplus
}
#endif

#endif /* MP_KERNELS_H */
