// fp64 CUDA-core throughput on this GPU (roofline denominators for the fp64 kernels):
// independent DFMA chains, and DMUL + DADD pairs (the reference-order scoring kernels).
//   nvcc -O3 -gencode arch=compute_100a,code=sm_100a -o fp64_probe scripts/fp64_probe.cu && ./fp64_probe
#include <cstdio>
#include <cuda_runtime.h>

template <bool FMA>
__global__ void chains(double* out, int iters, double a, double b) {
    double x[8];
#pragma unroll
    for (int i = 0; i < 8; ++i) x[i] = threadIdx.x * 1e-3 + i;
    for (int it = 0; it < iters; ++it) {
#pragma unroll
        for (int i = 0; i < 8; ++i) {
            if (FMA) x[i] = fma(x[i], a, b);
            else x[i] = __dadd_rn(__dmul_rn(x[i], a), b);
        }
    }
    double s = 0;
#pragma unroll
    for (int i = 0; i < 8; ++i) s += x[i];
    out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

int main() {
    int sms = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    const int blocks = sms * 8, threads = 256, iters = 4096;
    double* out;
    cudaMalloc(&out, sizeof(double) * blocks * threads);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    for (int mode = 0; mode < 2; ++mode) {
        for (int rep = 0; rep < 2; ++rep) {
            cudaEventRecord(e0);
            if (mode == 0) chains<true><<<blocks, threads>>>(out, iters, 0.999999, 1e-7);
            else chains<false><<<blocks, threads>>>(out, iters, 0.999999, 1e-7);
            cudaEventRecord(e1);
            cudaEventSynchronize(e1);
        }
        float ms = 0;
        cudaEventElapsedTime(&ms, e0, e1);
        const double terms = double(blocks) * threads * iters * 8;  // (x*a + b) terms
        printf("{\"%s\": {\"ms\": %.3f, \"tflops\": %.2f}}\n", mode == 0 ? "dfma" : "dmul_dadd", ms,
               2.0 * terms / (ms * 1e-3) / 1e12);
    }
    return 0;
}
