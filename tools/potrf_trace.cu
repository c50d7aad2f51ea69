#define TC_POTRF_TRACE 1
#include <cstdio>
#include <vector>
#include "../paper_2501_02483_b200/csrc/tc_kernels.cuh"
using namespace tc;
int main() {
    for (int nt : {120, 128, 160, 184}) {
        std::vector<double> h(nt * nt);
        for (int j = 0; j < nt; ++j) for (int i = 0; i < nt; ++i) h[j * nt + i] = (i == j) ? nt + 1.0 : 1.0 / (1 + i + j);
        double* d; cudaMalloc(&d, nt * nt * 8);
        int ntp = (nt + 7) & ~7; size_t sm = potrf_smem_bytes(ntp, true);
        cudaFuncSetAttribute(k_potrf, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
        PotrfArgs pa{}; pa.tile = d; pa.nt = nt; pa.in_smem = 1;
        float best = 1e9;
        for (int it = 0; it < 5; ++it) {
            cudaMemcpy(d, h.data(), nt * nt * 8, cudaMemcpyHostToDevice);
            cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
            cudaEventRecord(e0);
            k_potrf<<<1, kPotrfThreads, sm>>>(pa);
            cudaEventRecord(e1); cudaEventSynchronize(e1);
            float ms; cudaEventElapsedTime(&ms, e0, e1); if (ms < best) best = ms;
        }
        long long t[4096];
        cudaMemcpyFromSymbol(t, g_potrf_trace, sizeof(t));
        int NB = ntp / 8;
        long long t0 = t[1];
        printf("nt=%d k_potrf best %.1f us; per panel [chol_start chol_done next_solved] rel cycles\n", nt, best * 1e3);
        for (int K = 0; K < NB && K < 8; ++K) printf("  K=%2d %7lld %7lld %7lld\n", K, t[4*K+1]-t0, t[4*K+2]-t0, (K+1<NB)? t[4*K+3]-t0 : 0);
        printf("  last chol_done %lld cycles\n", t[4*(NB-1)+2]-t0);
    }
}
