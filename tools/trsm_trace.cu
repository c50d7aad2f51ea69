// TRSM strip timing: k_trsm<ROWS> on one nt x nt target (direct mode), per-panel clock trace of warp 0.
#define TC_TRSM_TRACE 1
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <vector>
#include "../paper_2501_02483_b200/csrc/tc_kernels.cuh"
using namespace tc;
int main(int argc, char** argv) {
    const int nt = argc > 1 ? atoi(argv[1]) : 128;
    std::vector<double> L(nt * nt, 0.0), B(nt * nt);
    for (int j = 0; j < nt; ++j)
        for (int i = j; i < nt; ++i) L[j * nt + i] = (i == j) ? 2.0 : 0.01 / (1 + i - j);
    for (int j = 0; j < nt; ++j)
        for (int i = 0; i < nt; ++i) B[j * nt + i] = 1.0 / (1 + i + 2 * j);
    double *dL, *dB;
    cudaMalloc(&dL, nt * nt * 8);
    cudaMalloc(&dB, nt * nt * 8);
    cudaMemcpy(dL, L.data(), nt * nt * 8, cudaMemcpyHostToDevice);
    const int ROWS = 64;
    size_t sm = trsm_smem_bytes<64>(nt);
    cudaFuncSetAttribute(k_trsm<64>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
    TrsmArgs ta{};
    ta.L = dL;
    ta.X = dB;
    ta.nt = nt;
    float best = 1e9;
    for (int it = 0; it < 10; ++it) {
        cudaMemcpy(dB, B.data(), nt * nt * 8, cudaMemcpyHostToDevice);
        cudaEvent_t e0, e1;
        cudaEventCreate(&e0);
        cudaEventCreate(&e1);
        cudaEventRecord(e0);
        k_trsm<64><<<dim3((nt + ROWS - 1) / ROWS, 1), 4 * ROWS, sm>>>(ta);
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        float ms;
        cudaEventElapsedTime(&ms, e0, e1);
        if (ms < best) best = ms;
    }
    std::vector<double> X(nt * nt);
    cudaMemcpy(X.data(), dB, nt * nt * 8, cudaMemcpyDeviceToHost);
    double err = 0;  // || X L^T - B ||_max
    for (int i = 0; i < nt; ++i)
        for (int j = 0; j < nt; ++j) {
            double s = 0;
            for (int c = 0; c <= j; ++c) s += X[c * nt + i] * L[c * nt + j];
            err = fmax(err, fabs(s - B[j * nt + i]));
        }
    long long t[256];
    cudaMemcpyFromSymbol(t, g_trsm_trace, sizeof(t));
    printf("nt=%d k_trsm<64> best %.2f us, max resid %.2e, %s\n", nt, best * 1e3, err, cudaGetErrorString(cudaGetLastError()));
    for (int K = 0; K < (nt + 7) / 8; ++K)
        printf("K=%2d gemm %5lld solve %5lld  next %5lld\n", K, t[3 * K + 1] - t[3 * K], t[3 * K + 2] - t[3 * K + 1],
               K + 1 < (nt + 7) / 8 ? t[3 * K + 3] - t[3 * K + 2] : 0);
}
