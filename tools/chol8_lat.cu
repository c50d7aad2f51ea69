// Isolated latency of chol8_regs / solve8_row (one warp), cycles per call.
#include <cstdio>
#include "../paper_2501_02483_b200/csrc/tc_kernels.cuh"
using namespace tc;
__global__ void k(double* out, long long* cyc, int mode) {
    __shared__ double D[8 * 12 * 2];
    const int lane = threadIdx.x & 31;
    for (int i = threadIdx.x; i < 8 * 12 * 2; i += blockDim.x) D[i] = (i % 13 == 0) ? 10.0 : 0.1;
    __syncthreads();
    double l[8][8], inv[8], acc = 0;
    if (threadIdx.x < 32) {
        long long t0 = clock64();
        for (int r = 0; r < 64; ++r) {
            chol8_regs(D + (r & 1) * 96, 12, 0, l, inv);
            acc += l[7][7];
            D[(r & 1) * 96 + 5] = acc * 1e-30 + 0.1;  // dependency between calls
            __syncwarp();
        }
        long long t1 = clock64();
        double x[8];
        for (int c = 0; c < 8; ++c) x[c] = D[c * 12 + (lane & 7)];
        long long t2 = clock64();
        for (int r = 0; r < 64; ++r) {
            solve8_row(x, l, inv);
            x[0] += acc * 1e-30;
        }
        long long t3 = clock64();
        if (lane == 0) {
            cyc[0] = (t1 - t0) / 64;
            cyc[1] = (t3 - t2) / 64;
        }
        out[lane] = acc + x[7];
        if (lane == 0) atomicExch((int*)&cyc[7], 1);
    } else if (mode == 1) {  // interference: DMMA + LDS loops until warp 0 is done
        __shared__ double S[2048];
        for (int i = threadIdx.x; i < 2048; i += blockDim.x) S[i] = 1e-3;
        double d0 = 0, d1 = 0;
        const int g = lane >> 2, q = lane & 3;
        int it = 0;
        while (*(volatile int*)&cyc[7] == 0 && it < 200000) {
            for (int u = 0; u < 16; ++u) {
                const double a = S[(u * 4 + q) * 12 + g + (threadIdx.x >> 5) * 100], b = S[(u * 4 + q) * 12 + g + 50];
                dmma(d0, d1, a, b);
            }
            ++it;
        }
        out[32 + threadIdx.x] = d0 + d1;
    } else if (mode == 2) {  // interference: spin loops on smem
        int it = 0;
        while (*(volatile int*)&cyc[7] == 0 && it < 20000000) ++it;
        out[32 + threadIdx.x] = it;
    }
}
int main() {
    double* o;
    long long* c;
    cudaMalloc(&o, 1024);
    cudaMallocManaged(&c, 64);
    for (int r = 0; r < 2; ++r) {
        k<<<1, 32>>>(o, c, 0);
        cudaDeviceSynchronize();
    }
    printf("chol8_regs %lld cycles/call, solve8_row %lld cycles/call (1 warp)\n", c[0], c[1]);
    const char* nm[] = {"7 idle", "7 DMMA+LDS", "7 spinning"};
    for (int y = 0; y < 3; ++y) {
        for (int r = 0; r < 2; ++r) {
            c[7] = 0;
            k<<<1, 256>>>(o, c, y);
            cudaDeviceSynchronize();
        }
    }
    for (int y = 0; y < 3; ++y) {
        c[7] = 0;
        k<<<1, 256>>>(o, c, y);
        cudaDeviceSynchronize();
        printf("chol8_regs %lld cycles/call, solve8_row %lld (%s)\n", c[0], c[1], nm[y]);
    }
}
