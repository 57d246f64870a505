// dadd_bench.cu -- dependent-chain latency and throughput of FP64 add on this GPU.
#include <cuda_runtime.h>
#include <cstdio>
__global__ void chain(double *out, long long *cyc, int iters, double a) {
    double s = threadIdx.x;
    long long t0 = clock64();
    for (int i = 0; i < iters; ++i) s = __dadd_rn(s, a);
    long long t1 = clock64();
    out[blockIdx.x * blockDim.x + threadIdx.x] = s;
    if (threadIdx.x == 0 && blockIdx.x == 0) *cyc = t1 - t0;
}
__global__ void chain_f32(float *out, long long *cyc, int iters, float a) {
    float s = threadIdx.x;
    long long t0 = clock64();
    for (int i = 0; i < iters; ++i) s = __fadd_rn(s, a);
    long long t1 = clock64();
    out[blockIdx.x * blockDim.x + threadIdx.x] = s;
    if (threadIdx.x == 0 && blockIdx.x == 0) *cyc = t1 - t0;
}
int main() {
    double *o; float *of; long long *c, h;
    cudaMalloc(&o, 1 << 24); cudaMalloc(&of, 1 << 24); cudaMalloc(&c, 8);
    const int it = 1 << 16;
    chain<<<1, 1>>>(o, c, it, 1e-3); cudaMemcpy(&h, c, 8, cudaMemcpyDeviceToHost);
    printf("DADD dependent latency: %.2f cycles\n", (double)h / it);
    chain_f32<<<1, 1>>>(of, c, it, 1e-3f); cudaMemcpy(&h, c, 8, cudaMemcpyDeviceToHost);
    printf("FADD dependent latency: %.2f cycles\n", (double)h / it);
    int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
    for (int tpb : {128, 512, 1024}) {
        chain<<<sms * 2, tpb>>>(o, c, it, 1e-3);
        cudaEventRecord(e0); chain<<<sms * 2, tpb>>>(o, c, it, 1e-3); cudaEventRecord(e1); cudaEventSynchronize(e1);
        float ms; cudaEventElapsedTime(&ms, e0, e1);
        printf("DADD throughput tpb %4d: %.1f Gadd/s (%.1f per SM per cycle @1.965GHz)\n", tpb,
               (double)sms * 2 * tpb * it / ms / 1e6, (double)2 * tpb * it / (ms * 1e-3 * 1.965e9));
    }
    return 0;
}
