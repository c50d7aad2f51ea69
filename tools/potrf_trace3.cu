// Per-step clock trace of potrf_body (diagonal warp + critical worker), nt from argv.
#define TC_POTRF_TRACE 1
#include <cstdio>
#include <cstdlib>
#include <vector>
#include "../paper_2501_02483_b200/csrc/tc_kernels.cuh"
using namespace tc;
int main(int argc, char** argv) {
    const int nt = argc > 1 ? atoi(argv[1]) : 120;
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
    long long t0 = t[5];  // chol8(0) done
    printf("nt=%d cycles rel. to chol8(0): diag[start gotready gemm solve rank8 chol8 pub] | crit worker of K+2 [gotdiag gemm solve+rank8 ready]\n", nt);
    for (int K = 0; K < NB; ++K) {
        printf("K=%2d", K);
        for (int x = 0; x < 7; ++x) printf(" %7lld", t[8 * K + x] ? t[8 * K + x] - t0 : -1);
        printf(" |");
        for (int x = 0; x < 4; ++x) printf(" %7lld", t[512 + 4 * K + x] ? t[512 + 4 * K + x] - t0 : -1);
        printf("\n");
    }
    printf("%s\n", cudaGetErrorString(cudaGetLastError()));
}
