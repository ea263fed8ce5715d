// ubench_fp64.cu — measured FP64 peaks on this B200 (DFMA pipe and the FP64 mma.sync / DMMA path),
// the roofline denominators of the binary64 (mp_dgesv) path.  nvcc -gencode arch=compute_100a,code=sm_100a
#include <cstdio>
#include <cuda_runtime.h>

__global__ void dfma_loop(double *out, int iters)
{
    double a[8], b = 1.0000001, c = 0.9999999;
#pragma unroll
    for (int i = 0; i < 8; ++i) a[i] = threadIdx.x + i;
    for (int it = 0; it < iters; ++it) {
#pragma unroll
        for (int i = 0; i < 8; ++i) a[i] = fma(a[i], b, c);
    }
    double s = 0;
#pragma unroll
    for (int i = 0; i < 8; ++i) s += a[i];
    if (s == 12345.0) out[0] = s;
}

template <int SHAPE>
__global__ void dmma_loop(double *out, int iters)
{
    // SHAPE 0: m8n8k4 (256 FMA / warp-instr); 1: m16n8k4 (512); 2: m16n8k8 (1024); 3: m16n8k16 (2048)
    double acc[4][4] = {};
    double a[8], b[4];
#pragma unroll
    for (int i = 0; i < 8; ++i) a[i] = 1.0 + 1e-9 * (threadIdx.x + i);
#pragma unroll
    for (int i = 0; i < 4; ++i) b[i] = 1.0 - 1e-9 * (threadIdx.x + i);
    for (int it = 0; it < iters; ++it) {
#pragma unroll
        for (int j = 0; j < 4; ++j) {
            if constexpr (SHAPE == 0) {
                asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
                             : "+d"(acc[j][0]), "+d"(acc[j][1]) : "d"(a[j]), "d"(b[j]));
            } else if constexpr (SHAPE == 1) {
                asm volatile("mma.sync.aligned.m16n8k4.row.col.f64.f64.f64.f64 {%0,%1,%2,%3}, {%4,%5}, {%6}, {%0,%1,%2,%3};"
                             : "+d"(acc[j][0]), "+d"(acc[j][1]), "+d"(acc[j][2]), "+d"(acc[j][3])
                             : "d"(a[j]), "d"(a[j + 4]), "d"(b[j]));
            } else if constexpr (SHAPE == 2) {
                asm volatile("mma.sync.aligned.m16n8k8.row.col.f64.f64.f64.f64 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, {%0,%1,%2,%3};"
                             : "+d"(acc[j][0]), "+d"(acc[j][1]), "+d"(acc[j][2]), "+d"(acc[j][3])
                             : "d"(a[0]), "d"(a[1]), "d"(a[2]), "d"(a[3]), "d"(b[j]), "d"(b[(j + 1) & 3]));
            } else {
                asm volatile("mma.sync.aligned.m16n8k16.row.col.f64.f64.f64.f64 {%0,%1,%2,%3}, {%4,%5,%6,%7,%8,%9,%10,%11}, {%12,%13,%14,%15}, {%0,%1,%2,%3};"
                             : "+d"(acc[j][0]), "+d"(acc[j][1]), "+d"(acc[j][2]), "+d"(acc[j][3])
                             : "d"(a[0]), "d"(a[1]), "d"(a[2]), "d"(a[3]), "d"(a[4]), "d"(a[5]), "d"(a[6]), "d"(a[7]),
                               "d"(b[0]), "d"(b[1]), "d"(b[2]), "d"(b[3]));
            }
        }
    }
    double s = 0;
#pragma unroll
    for (int j = 0; j < 4; ++j)
#pragma unroll
        for (int i = 0; i < 4; ++i) s += acc[j][i];
    if (s == 12345.0) out[0] = s;
}

template <typename F>
double run(F kern, int blocks, int threads, int iters, double flops_per_thread_iter)
{
    double *out;
    cudaMalloc(&out, 8);
    kern<<<blocks, threads>>>(out, 10);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    cudaEventRecord(e0);
    kern<<<blocks, threads>>>(out, iters);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    cudaFree(out);
    return flops_per_thread_iter * iters * (double)blocks * threads / (ms * 1e-3) / 1e12;
}

int main()
{
    int sms;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    int clk;
    cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
    printf("sms %d clock %d kHz\n", sms, clk);
    for (int w : {4, 8, 16}) {
        double t = run(dfma_loop, sms * 4, 32 * w, 200000, 16.0);
        printf("DFMA  %2d warps/CTA x 4 CTA/SM: %.2f TFLOP/s\n", w, t);
    }
    for (int w : {4, 8, 16}) {
        printf("DMMA m8n8k4   %2d warps x4: %.2f TFLOP/s\n", w, run(dmma_loop<0>, sms * 4, 32 * w, 20000, 4 * 2.0 * 256 / 32));
        printf("DMMA m16n8k4  %2d warps x4: %.2f TFLOP/s\n", w, run(dmma_loop<1>, sms * 4, 32 * w, 20000, 4 * 2.0 * 512 / 32));
        printf("DMMA m16n8k8  %2d warps x4: %.2f TFLOP/s\n", w, run(dmma_loop<2>, sms * 4, 32 * w, 20000, 4 * 2.0 * 1024 / 32));
        printf("DMMA m16n8k16 %2d warps x4: %.2f TFLOP/s\n", w, run(dmma_loop<3>, sms * 4, 32 * w, 10000, 4 * 2.0 * 2048 / 32));
    }
    cudaError_t e = cudaGetLastError();
    printf("err: %s\n", cudaGetErrorString(e));
    return 0;
}
