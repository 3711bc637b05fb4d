// Developer microbenchmark (not product): FP64 DFMA dependent-chain latency
// and throughput vs warps per scheduler on this GPU.
#include <cstdio>
#include <cuda_runtime.h>
__global__ void chain(double *out, int iters, double a, double b, long long *cyc)
{
    double x = threadIdx.x * 1e-9;
    long long t0 = clock64();
    for (int i = 0; i < iters; i++) {
#pragma unroll
        for (int k = 0; k < 32; k++) x = fma(x, a, b);
    }
    long long t1 = clock64();
    if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
    if (x == 1.2345) out[0] = x;
}
template <int ILP>
__global__ void ilp(double *out, int iters, double a, double b)
{
    double x[ILP];
#pragma unroll
    for (int j = 0; j < ILP; j++) x[j] = threadIdx.x * 1e-9 + j;
    for (int i = 0; i < iters; i++) {
#pragma unroll
        for (int k = 0; k < 16; k++)
#pragma unroll
            for (int j = 0; j < ILP; j++) x[j] = fma(x[j], a, b);
    }
    double s = 0;
#pragma unroll
    for (int j = 0; j < ILP; j++) s += x[j];
    if (s == 1.2345) out[0] = s;
}
int main()
{
    double *d; long long *c; cudaMalloc(&d, 8); cudaMalloc(&c, 8 * 1024);
    chain<<<1, 32>>>(d, 1000, 0.999, 1e-9, c); cudaDeviceSynchronize();
    chain<<<1, 32>>>(d, 10000, 0.999, 1e-9, c);
    long long h; cudaMemcpy(&h, c, 8, cudaMemcpyDeviceToHost);
    printf("DFMA dependent latency: %.2f cycles\n", (double)h / (10000.0 * 32));
    cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
    int sms = 148;
    for (int wps = 1; wps <= 8; wps *= 2) {
        // wps warps per scheduler -> 4*wps warps per SM -> block of 128*wps threads, 1 block per SM
        float ms;
        int it = 2000;
        ilp<1><<<sms, 128 * wps>>>(d, 10, 0.999, 1e-9);
        cudaEventRecord(e0); ilp<1><<<sms, 128 * wps>>>(d, it, 0.999, 1e-9); cudaEventRecord(e1); cudaEventSynchronize(e1);
        cudaEventElapsedTime(&ms, e0, e1);
        double fl1 = 2.0 * 16 * it * 128.0 * wps * sms;
        cudaEventRecord(e0); ilp<2><<<sms, 128 * wps>>>(d, it, 0.999, 1e-9); cudaEventRecord(e1); cudaEventSynchronize(e1);
        float ms2; cudaEventElapsedTime(&ms2, e0, e1);
        cudaEventRecord(e0); ilp<4><<<sms, 128 * wps>>>(d, it, 0.999, 1e-9); cudaEventRecord(e1); cudaEventSynchronize(e1);
        float ms4; cudaEventElapsedTime(&ms4, e0, e1);
        printf("warps/scheduler %d: ILP1 %.1f TF  ILP2 %.1f TF  ILP4 %.1f TF\n", wps, fl1 / ms / 1e9, 2 * fl1 / ms2 / 1e9, 4 * fl1 / ms4 / 1e9);
    }
    return 0;
}
