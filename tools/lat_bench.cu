// Dependent-chain latencies on the B200 (one thread): DADD (__dadd_rn), DMUL, and a
// shared-memory load feeding a DADD -- the numbers behind the in-order folds (wide rows,
// exact sequential sums).  nvcc -gencode arch=compute_100a,code=sm_100a -O3 -fmad=false
#include <cstdio>
#include <cuda_runtime.h>

__global__ void k_lat(double *out, long long *cyc, int iters, double a) {
    __shared__ double sm[1024];
    for (int i = threadIdx.x; i < 1024; i += blockDim.x) sm[i] = 1e-20 * i;
    __syncthreads();
    if (threadIdx.x) return;
    double s = a;
    long long t0 = clock64();
    for (int i = 0; i < iters; ++i) s = __dadd_rn(s, a);
    long long t1 = clock64();
    double m = a;
    for (int i = 0; i < iters; ++i) m = __dmul_rn(m, 1.0000001);
    long long t2 = clock64();
    double f = 0.0;
    for (int i = 0; i < iters; ++i) f = __dadd_rn(f, sm[i & 1023]);
    long long t3 = clock64();
    // dependent smem pointer chase through an index (LDS latency)
    int idx = 0;
    int *smi = reinterpret_cast<int *>(sm);
    for (int i = 0; i < 1024; ++i) smi[i] = (i + 1) & 1023;
    long long t4 = clock64();
    for (int i = 0; i < iters; ++i) idx = smi[idx];
    long long t5 = clock64();
    out[0] = s + m + f + idx;
    cyc[0] = t1 - t0;
    cyc[1] = t2 - t1;
    cyc[2] = t3 - t2;
    cyc[3] = t5 - t4;
}

int main() {
    double *d;
    long long *c, h[4];
    cudaMalloc(&d, 8);
    cudaMalloc(&c, 32);
    const int it = 100000;
    k_lat<<<1, 32>>>(d, c, it, 1.5);
    k_lat<<<1, 32>>>(d, c, it, 1.5);
    cudaMemcpy(h, c, 32, cudaMemcpyDeviceToHost);
    printf("cycles per dependent op: DADD %.2f  DMUL %.2f  DADD(s, LDS[i]) %.2f  LDS chase %.2f\n",
           (double)h[0] / it, (double)h[1] / it, (double)h[2] / it, (double)h[3] / it);
    return 0;
}
