// Phase timing of the POTRF body (clock64) on one random SPD tile.
#include <cstdio>
#include <vector>
#include <cmath>
#include "../paper_2501_02483_b200/csrc/tc_kernels.cuh"
using namespace tc;

template <int NTH>
__global__ void k_probe(double* A, int nt, long long* tl) {
    extern __shared__ __align__(16) double smem[];
    __shared__ int s_info;
    const int ntp = (nt + 7) & ~7, ld = pad_ld(ntp);
    double* M = smem; double* s_inv = smem + (size_t)ntp * ld;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5, g = lane >> 2, q = lane & 3;
    constexpr int NW = NTH / 32;
    long long t0 = clock64();
    for (int e = tid; e < ntp * ntp; e += NTH) { int c = e / ntp, r = e % ntp; M[c * ld + r] = (c < nt && r < nt) ? A[c * nt + r] : (r == c); }
    if (tid == 0) s_info = -1;
    __syncthreads();
    long long t1 = clock64();
    long long tg = 0, tc8 = 0, tb1 = 0, ttr = 0, tb2 = 0;
    const int NB = ntp / 8;
    for (int K = 0; K < NB; ++K) {
        const int c0 = 8 * K, owner = K % NW;
        long long a = clock64();
        if (K > 0) {
            int rb = K + ((warp - K % NW) + NW) % NW;
            for (; rb < NB; rb += NW) { panel_gemm8(M, ld, 8 * rb, c0, g, q); if (rb == K) __syncwarp(); if (rb == K && warp == owner) break; }
        }
        long long b = clock64();
        if (warp == owner) {
            double l[8][8], inv[8];
            int bad = chol8_regs(M, ld, c0, l, inv);
#pragma unroll
            for (int i = 0; i < 8; ++i) if (lane == i) {
#pragma unroll
                for (int c = 0; c <= i; ++c) M[(c0 + c) * ld + c0 + i] = l[i][c];
                s_inv[c0 + i] = inv[i]; }
            if (bad >= 0 && lane == 0) s_info = bad;
            if (K > 0) for (int rb = K + NW; rb < NB; rb += NW) panel_gemm8(M, ld, 8 * rb, c0, g, q);
        }
        long long c = clock64();
        __syncthreads();
        long long d = clock64();
        long long s0 = 0, s1 = 0, s2 = 0, s3 = 0, s4 = 0;
        if (c0 + 8 + tid < ntp) {
            s0 = clock64();
            double l[8][8], inv[8];
#pragma unroll
            for (int i = 0; i < 8; ++i) { inv[i] = s_inv[c0 + i];
#pragma unroll
                for (int cc = 0; cc < i; ++cc) l[i][cc] = M[(c0 + cc) * ld + c0 + i]; }
            s1 = clock64();
            for (int r = c0 + 8 + tid; r < ntp; r += NTH) {
                double x[8];
#pragma unroll
                for (int cc = 0; cc < 8; ++cc) x[cc] = M[(c0 + cc) * ld + r];
                s2 = clock64();
                solve8_row(x, l, inv);
                s3 = clock64();
#pragma unroll
                for (int cc = 0; cc < 8; ++cc) M[(c0 + cc) * ld + r] = x[cc];
                s4 = clock64();
            }
        }
        if (tid == 0 && s0) { tl[9] += s0 - d; tl[10] += s1 - s0; tl[11] += s2 - s1; tl[12] += s3 - s2; tl[13] += s4 - s3; tl[14] += clock64() - s4; }
        long long e = clock64();
        __syncthreads();
        long long f = clock64();
        if (warp == owner) { tg += b - a; tc8 += c - b; }
        tb1 += d - c; ttr += e - d; tb2 += f - e;
    }
    long long t2 = clock64();
    for (int e = tid; e < nt * nt; e += NTH) { int c = e / nt, r = e % nt; A[c * nt + r] = r >= c ? M[c * ld + r] : 0.0; }
    __syncthreads();
    long long t3 = clock64();
    if (tid == 0) { tl[0] = t1 - t0; tl[1] = t2 - t1; tl[2] = t3 - t2; tl[3] = tg; tl[4] = tc8; tl[5] = tb1; tl[6] = ttr; tl[7] = tb2; tl[8] = s_info; }
}

int main() {
    for (int nt : {120, 160}) {
        std::vector<double> h(nt * nt);
        for (int j = 0; j < nt; ++j) for (int i = 0; i < nt; ++i) h[j * nt + i] = (i == j) ? nt + 1.0 : 1.0 / (1 + i + j);
        double* d; long long* tl; cudaMalloc(&d, nt * nt * 8); cudaMalloc(&tl, 16 * 8); cudaMemset(tl, 0, 128);
        int ntp = (nt + 7) & ~7; size_t sm = (size_t)ntp * pad_ld(ntp) * 8 + ntp * 8;
        cudaFuncSetAttribute(k_probe<256>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
        long long ht[16];
        for (int it = 0; it < 3; ++it) {
            cudaMemcpy(d, h.data(), nt * nt * 8, cudaMemcpyHostToDevice);
            cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
            cudaEventRecord(e0);
            k_probe<256><<<1, 256, sm>>>(d, nt, tl);
            cudaEventRecord(e1); cudaEventSynchronize(e1);
            float ms; cudaEventElapsedTime(&ms, e0, e1);
            cudaMemcpy(ht, tl, 16 * 8, cudaMemcpyDeviceToHost);
            printf("nt=%d %.1f us | load %lld body %lld wb %lld | owner gemm %lld chol8 %lld | bar1 %lld trsm %lld bar2 %lld | info %lld | entry %lld lpre %lld xld %lld solve %lld st %lld tail %lld | err %s\n",
                   nt, ms * 1e3, ht[0], ht[1], ht[2], ht[3], ht[4], ht[5], ht[6], ht[7], ht[8], ht[9], ht[10], ht[11], ht[12], ht[13], ht[14], cudaGetErrorString(cudaGetLastError()));
            cudaMemset(tl, 0, 128);
        }
        // real kernel timing
        PotrfArgs pa{}; pa.tile = d; pa.nt = nt; pa.in_smem = 1;
        cudaFuncSetAttribute(k_potrf, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
        for (int it = 0; it < 3; ++it) {
            cudaMemcpy(d, h.data(), nt * nt * 8, cudaMemcpyHostToDevice);
            cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
            cudaEventRecord(e0);
            k_potrf<<<1, kPotrfThreads, sm>>>(pa);
            cudaEventRecord(e1); cudaEventSynchronize(e1);
            float ms; cudaEventElapsedTime(&ms, e0, e1);
            printf("k_potrf nt=%d %.1f us\n", nt, ms * 1e3);
        }
    }
    return 0;
}
