// Per-step clock trace of potrf_body (diagonal warp: after GEMM / after chol8+publish / after solve+rank8).
#define TC_POTRF_TRACE 1
#include <cstdio>
#include <cstdlib>
#include <vector>
#include "../paper_2501_02483_b200/csrc/tc_kernels.cuh"
using namespace tc;
int main(int argc, char** argv) {
    const int nt = argc > 1 ? atoi(argv[1]) : 128;
    std::vector<double> h(nt * nt);
    for (int j = 0; j < nt; ++j)
        for (int i = 0; i < nt; ++i) h[j * nt + i] = (i == j) ? nt + 1.0 : 1.0 / (1 + i + j);
    double* d;
    cudaMalloc(&d, nt * nt * 8);
    int ntp = (nt + 7) & ~7;
    size_t sm = potrf_smem_bytes(ntp, true);
    cudaFuncSetAttribute(k_potrf, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
    PotrfArgs pa{};
    pa.tile = d;
    pa.nt = nt;
    pa.in_smem = 1;
    for (int it = 0; it < 3; ++it) {
        cudaMemcpy(d, h.data(), nt * nt * 8, cudaMemcpyHostToDevice);
        k_potrf<<<1, kPotrfThreads, sm>>>(pa);
        cudaDeviceSynchronize();
    }
    std::vector<long long> t(4096);
    cudaMemcpyFromSymbol(t.data(), g_potrf_trace, 2048 * 8);
    const int NB = ntp / 8;
    long long t0 = t[0];
    printf("nt=%d diag warp cycles: [start, got rowdone(K+1), gemm done, chol8+pub done, solve+rank8 done] | worker of K+2 [got diag(K), rowdone]\n", nt);
    for (int K = 0; K < NB; ++K)
        printf("K=%2d %7lld %7lld %7lld %7lld %7lld | %7lld %7lld\n", K, t[4 * K] - t0, t[1024 + K] ? t[1024 + K] - t0 : -1,
               t[4 * K + 1] - t0, t[4 * K + 2] - t0, t[4 * K + 3] - t0,
               t[512 + 4 * K] ? t[512 + 4 * K] - t0 : -1, t[512 + 4 * K + 1] ? t[512 + 4 * K + 1] - t0 : -1);
    printf("%s\n", cudaGetErrorString(cudaGetLastError()));
}
