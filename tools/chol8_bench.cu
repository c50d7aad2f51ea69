#include <cstdio>
#include "../paper_2501_02483_b200/csrc/tc_kernels.cuh"
using namespace tc;
__device__ __forceinline__ int chol8_nort(const double* M, int ld, int c0, double (&l)[8][8], double (&inv)[8]) {
#pragma unroll
    for (int i = 0; i < 8; ++i)
#pragma unroll
        for (int c = 0; c <= i; ++c) l[i][c] = M[(size_t)(c0 + c) * ld + c0 + i];
    int bad = -1;
#pragma unroll
    for (int j = 0; j < 8; ++j) {
        const double piv = l[j][j];
        if (piv <= 0.0 && bad < 0) bad = j;
        const double r = rsqrt(piv);
        inv[j] = r;
        l[j][j] = piv * r;
#pragma unroll
        for (int i = j + 1; i < 8; ++i) l[i][j] *= r;
#pragma unroll
        for (int c = j + 1; c < 8; ++c)
#pragma unroll
            for (int i = c; i < 8; ++i) l[i][c] -= l[i][j] * l[c][j];
    }
    return bad;
}
__global__ void kb(double* out, long long* t, int reps) {
    __shared__ double M[64 * 12];
    int lane = threadIdx.x;
    for (int i = lane; i < 64 * 12; i += 32) M[i] = 0;
    __syncwarp();
    if (lane < 8) for (int c = 0; c < 8; ++c) M[c * 12 + lane] = (lane == c) ? 10.0 : 0.5;
    __syncwarp();
    double l[8][8], inv[8], acc = 0;
    long long a = clock64();
    for (int r = 0; r < reps; ++r) { int b = chol8_regs(M, 12, 0, l, inv); acc += l[7][7] + b; __syncwarp(); }
    long long b = clock64();
    for (int r = 0; r < reps; ++r) { int bb = chol8_nort(M, 12, 0, l, inv); acc += l[7][7] + bb; __syncwarp(); }
    long long c = clock64();
    double x[8];
    for (int r = 0; r < reps; ++r) {
        for (int i = 0; i < 8; ++i) x[i] = M[i * 12 + lane % 8] + r;
        solve8_row(x, l, inv); acc += x[7];
    }
    long long d = clock64();
    double z = 1.0 + lane;
    for (int r = 0; r < reps; ++r) { z = rsqrt(z + 1.0); }
    long long e = clock64();
    double w[8] = {1,2,3,4,5,6,7,8};
    for (int r = 0; r < reps; ++r) {
#pragma unroll
        for (int i = 0; i < 8; ++i) w[i] = fma(w[i], 0.999, 1e-3);
    }
    long long f = clock64();
    if (lane == 0) { t[0] = (b - a) / reps; t[1] = (c - b) / reps; t[2] = (d - c) / reps; t[3] = (e - d) / reps; t[4] = (f - e) / reps; }
    out[lane] = acc + z + w[0] + w[7];
}
int main() {
    double* o; long long* t; cudaMalloc(&o, 256); cudaMalloc(&t, 64);
    kb<<<1, 32>>>(o, t, 100); kb<<<1, 32>>>(o, t, 1000); cudaDeviceSynchronize();
    long long h[8]; cudaMemcpy(h, t, 64, cudaMemcpyDeviceToHost);
    printf("cycles per call: chol8_regs %lld chol8_no_early_return %lld solve8_row %lld rsqrt_chain %lld 8xdfma_indep %lld\n", h[0], h[1], h[2], h[3], h[4]);
}
