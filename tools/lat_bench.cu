// Dependent-chain latencies (cycles) of DFMA, DMUL, rsqrt.approx.f64 (MUFU.RSQ64H), DMMA, LDS.64.
#include <cstdio>
__global__ void k(double* out, long long* cyc, double x0) {
    double x = x0, y = 1.0000001;
    long long t0, t1;
    // DFMA chain
    t0 = clock64();
#pragma unroll 1
    for (int i = 0; i < 128; ++i) {
#pragma unroll
 for (int u = 0; u < 8; ++u) x = fma(x, y, 1e-9);
}
    t1 = clock64();
    cyc[0] = (t1 - t0);
    // DMUL chain
    t0 = clock64();
#pragma unroll 1
    for (int i = 0; i < 128; ++i) {
#pragma unroll
 for (int u = 0; u < 8; ++u) x = x * y;
}
    t1 = clock64();
    cyc[1] = (t1 - t0);
    // rsqrt chain
    t0 = clock64();
#pragma unroll 1
    for (int i = 0; i < 128; ++i) {
#pragma unroll
 for (int u = 0; u < 8; ++u) asm volatile("rsqrt.approx.ftz.f64 %0, %1;" : "=d"(x) : "d"(x));
}
    t1 = clock64();
    cyc[2] = (t1 - t0);
    // DMMA chain (accumulator dependency)
    double d0 = 0, d1 = 0;
    t0 = clock64();
#pragma unroll 1
    for (int i = 0; i < 1024; ++i)
#pragma unroll
        for (int u = 0; u < 1; ++u) asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
                     : "+d"(d0), "+d"(d1) : "d"(x), "d"(y));
    t1 = clock64();
    cyc[3] = (t1 - t0);
    // LDS chain
    __shared__ double sh[256];
    for (int i = threadIdx.x; i < 256; i += 32) sh[i] = 0.0;
    __syncwarp();
    int idx = threadIdx.x;
    t0 = clock64();
#pragma unroll 1
    for (int i = 0; i < 128; ++i) {
#pragma unroll
 for (int u = 0; u < 8; ++u) idx = (int)sh[idx & 255] + threadIdx.x;
}
    t1 = clock64();
    cyc[4] = (t1 - t0);
    // empty loop overhead
    int z = threadIdx.x;
    t0 = clock64();
#pragma unroll 1
    for (int i = 0; i < 1024; ++i) z = z * 3 + 1;
    t1 = clock64();
    cyc[5] = (t1 - t0);
    out[threadIdx.x] = x + d0 + d1 + idx + z;
}
int main() {
    double* o;
    long long* c;
    cudaMalloc(&o, 256);
    cudaMallocManaged(&c, 64);
    for (int r = 0; r < 2; ++r) {
        k<<<1, 32>>>(o, c, 1.5);
        cudaDeviceSynchronize();
    }
    const char* nm[] = {"DFMA", "DMUL", "RSQ64", "DMMA", "LDS(dep)", "IMAD loop"};
    for (int i = 0; i < 6; ++i) printf("%-10s %.1f cycles/iter\n", nm[i], c[i] / 1024.0);
}
