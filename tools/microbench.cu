// Latency microbenchmarks for the POTRF critical path (sm_100a).
#include <cstdio>
#include <cuda_runtime.h>
__device__ __forceinline__ void dmma(double& d0, double& d1, double a, double b) {
    asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n" : "+d"(d0), "+d"(d1) : "d"(a), "d"(b));
}
__global__ void k_lat(long long* out, double seed, int n) {
    double a = seed + threadIdx.x * 1e-9, b = seed * 0.5, d0 = 0, d1 = 0;
    long long t0 = clock64();
    for (int i = 0; i < n; ++i) dmma(d0, d1, a, b);           // dependent chain
    long long t1 = clock64();
    double x = seed + 2.0;
    for (int i = 0; i < n; ++i) x = rsqrt(x) + 1.5;
    long long t2 = clock64();
    double y = seed + 2.0;
    for (int i = 0; i < n; ++i) y = sqrt(y) + 1.5;
    long long t3 = clock64();
    double z = seed + 2.0;
    for (int i = 0; i < n; ++i) z = 1.0 / z + 1.5;
    long long t4 = clock64();
    double w = seed;
    for (int i = 0; i < n; ++i) w = fma(w, 0.999, 1e-3);
    long long t5 = clock64();
    double v = seed;
    for (int i = 0; i < n; ++i) v = __shfl_sync(0xffffffffu, v, (threadIdx.x + 1) & 31) + 1.0;
    long long t6 = clock64();
    __shared__ double sm[256];
    sm[threadIdx.x] = seed;
    __syncthreads();
    long long t7 = clock64();
    for (int i = 0; i < n; ++i) __syncthreads();
    long long t8 = clock64();
    volatile double* vs = sm;
    double u = 0;
    int idx = threadIdx.x;
    for (int i = 0; i < n; ++i) { u += vs[idx]; idx = (idx + (int)u) & 255; }
    long long t9 = clock64();
    if (threadIdx.x == 0) {
        out[0] = (t1 - t0) / n; out[1] = (t2 - t1) / n; out[2] = (t3 - t2) / n; out[3] = (t4 - t3) / n;
        out[4] = (t5 - t4) / n; out[5] = (t6 - t5) / n; out[6] = (t8 - t7) / n; out[7] = (t9 - t8) / n;
    }
    if (d0 + x + y + z + w + v + u == 1234.5) out[9] = 1;
}
int main() {
    long long* d; cudaMalloc(&d, 16 * 8);
    long long h[16];
    for (int threads : {32, 256}) {
        k_lat<<<1, threads>>>(d, 1.0, 1000);
        k_lat<<<1, threads>>>(d, 1.0, 1000);
        cudaMemcpy(h, d, 16 * 8, cudaMemcpyDeviceToHost);
        printf("threads=%d cycles/op: dmma_chain %lld rsqrt %lld sqrt %lld div %lld dfma %lld shfl %lld syncthreads %lld lds %lld\n",
               threads, h[0], h[1], h[2], h[3], h[4], h[5], h[6], h[7]);
    }
    return 0;
}
