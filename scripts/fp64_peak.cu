// FP64 DFMA throughput of one B200 ("FP64 peak is not in
// MEASURED_PEAKS.json; measure it with a DFMA microbenchmark"). Each thread runs
// 8 independent dependent-FMA chains; grid = SMs x 8 CTAs of 256 threads.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o scripts/_fp64_peak scripts/fp64_peak.cu
#include <cstdio>
#include <cuda_runtime.h>

__global__ void __launch_bounds__(256) k_dfma(double* out, int iters, double a, double b) {
    double x[8];
#pragma unroll
    for (int i = 0; i < 8; ++i) x[i] = threadIdx.x * 1e-3 + i;
    for (int it = 0; it < iters; ++it) {
#pragma unroll
        for (int i = 0; i < 8; ++i) x[i] = fma(x[i], a, b);
    }
    double s = 0.0;
#pragma unroll
    for (int i = 0; i < 8; ++i) s += x[i];
    if (s == 1234.5) out[0] = s; // keeps the chains live
}

int main() {
    int dev = 0, sms = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    double* out;
    cudaMalloc(&out, sizeof(double));
    const int blocks = sms * 8, threads = 256, iters = 1 << 14;
    k_dfma<<<blocks, threads>>>(out, 256, 0.999999, 1e-7); // warm-up
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    float best = 1e30f;
    for (int rep = 0; rep < 5; ++rep) {
        cudaEventRecord(e0);
        k_dfma<<<blocks, threads>>>(out, iters, 0.999999, 1e-7);
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        float ms = 0;
        cudaEventElapsedTime(&ms, e0, e1);
        best = ms < best ? ms : best;
    }
    const double flops = 2.0 * 8.0 * iters * static_cast<double>(blocks) * threads;
    printf("fp64_dfma_tflops: %.3f\nsms: %d\nms: %.3f\n", flops / (best * 1e-3) / 1e12, sms, best);
    return cudaGetLastError() == cudaSuccess ? 0 : 1;
}
