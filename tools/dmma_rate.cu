// DMMA issue-rate microbenchmark: cycles per DMMA for 1..8 warps, register vs smem operands.
#include <cstdio>
#include <cuda_runtime.h>
__device__ __forceinline__ void dmma(double& d0, double& d1, double a, double b) {
    asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n" : "+d"(d0), "+d"(d1) : "d"(a), "d"(b));
}
template <int NACC, bool SMEM>
__global__ void k(long long* out, double* sink, int iters, int active_warps) {
    __shared__ double s[12 * 128];
    for (int i = threadIdx.x; i < 12 * 128; i += blockDim.x) s[i] = 1.0 + i * 1e-6;
    __syncthreads();
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, g = lane >> 2, q = lane & 3;
    if (warp >= active_warps) return;
    double acc[NACC][2];
    for (int u = 0; u < NACC; ++u) acc[u][0] = acc[u][1] = 0;
    double a = 1.0 + lane * 1e-3, b = 2.0 - lane * 1e-3;
    long long t0 = clock64();
    for (int it = 0; it < iters; ++it) {
#pragma unroll
        for (int u = 0; u < NACC; ++u) {
            double av = a, bv = b;
            if (SMEM) {
                av = s[((it * 4 + q) % 96) * 12 + g + (u & 3) * 0];
                bv = s[((it * 4 + q + 8) % 96) * 12 + g];
            }
            dmma(acc[u][0], acc[u][1], av, bv);
        }
    }
    long long t1 = clock64();
    double t = 0;
    for (int u = 0; u < NACC; ++u) t += acc[u][0] + acc[u][1];
    sink[threadIdx.x] = t;
    if (lane == 0) out[warp] = (t1 - t0);
}
template <int NACC, bool SMEM>
void run(const char* name, int warps, int blocks) {
    long long* d; double* sink; cudaMalloc(&d, 64 * 8); cudaMalloc(&sink, 1024 * 8);
    int iters = 2000;
    k<NACC, SMEM><<<blocks, 256>>>(d, sink, iters, warps);
    k<NACC, SMEM><<<blocks, 256>>>(d, sink, iters, warps);
    cudaDeviceSynchronize();
    long long h[8]; cudaMemcpy(h, d, 8 * 8, cudaMemcpyDeviceToHost);
    printf("%-10s nacc=%d warps=%d blocks=%d: cycles/DMMA per warp %.1f\n", name, NACC, warps, blocks, (double)h[0] / (iters * NACC));
}
int main() {
    for (int w : {1, 2, 4, 8}) run<8, false>("regs", w, 1);
    for (int w : {1, 4}) run<4, false>("regs", w, 1);
    for (int w : {1, 4}) run<1, false>("regs", w, 1);
    for (int w : {1, 4, 8}) run<8, true>("smem", w, 1);
    run<8, false>("regs", 4, 148);
    run<8, false>("regs", 8, 296);
    return 0;
}
