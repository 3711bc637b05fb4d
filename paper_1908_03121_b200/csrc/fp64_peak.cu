// fp64_peak.cu -- measured FP64 roofline denominator (bench evidence only).
//
// MEASURED_PEAKS.json carries HBM and bf16 peaks but no FP64 figure; the
// stencil FMM kernels are FP64-pipe bound, so bench.py measures the FP64 DFMA
// throughput of this B200 with this kernel: every thread runs 8 independent
// DFMA chains (enough ILP to cover the pipe latency), 2 FLOP per DFMA, grid =
// 148 SMs x 8 CTAs x 256 threads, timed with CUDA events by the caller.
#include <cstdint>
#include <cuda_runtime.h>

__global__ void __launch_bounds__(256) dfma_peak_kernel(double *out, int iters, double a, double b)
{
    double x0 = threadIdx.x * 1e-7, x1 = x0 + 1e-3, x2 = x0 + 2e-3, x3 = x0 + 3e-3;
    double x4 = x0 + 4e-3, x5 = x0 + 5e-3, x6 = x0 + 6e-3, x7 = x0 + 7e-3;
    for (int i = 0; i < iters; i++) {
#pragma unroll
        for (int k = 0; k < 16; k++) {
            x0 = fma(x0, a, b); x1 = fma(x1, a, b); x2 = fma(x2, a, b); x3 = fma(x3, a, b);
            x4 = fma(x4, a, b); x5 = fma(x5, a, b); x6 = fma(x6, a, b); x7 = fma(x7, a, b);
        }
    }
    double s = x0 + x1 + x2 + x3 + x4 + x5 + x6 + x7;
    if (s == 12345.678) out[threadIdx.x] = s;   // keep the chains alive
}

// launches the kernel `reps` times on `stream`; returns flops per launch
extern "C" double octo_fp64_peak_launch(void *stream, int blocks, int iters, int reps)
{
    static double *d = nullptr;
    if (!d) cudaMalloc(&d, 256 * sizeof(double));
    for (int r = 0; r < reps; r++)
        dfma_peak_kernel<<<blocks, 256, 0, (cudaStream_t)stream>>>(d, iters, 0.9999999, 1e-9);
    return 2.0 * 8 * 16 * (double)iters * 256.0 * (double)blocks;
}
