#define TC_POTRF_TRACE 1
#include <cstdio>
#include <vector>
#include "../paper_2501_02483_b200/csrc/tc_kernels.cuh"
using namespace tc;
int main() {
    for (int nt : {120, 160}) {
        std::vector<double> h(nt * nt);
        for (int j = 0; j < nt; ++j) for (int i = 0; i < nt; ++i) h[j * nt + i] = (i == j) ? nt + 1.0 : 1.0 / (1 + i + j);
        double* d; cudaMalloc(&d, nt * nt * 8);
        int ntp = (nt + 7) & ~7; size_t sm = (size_t)ntp * pad_ld(ntp) * 8 + ntp * 8;
        cudaFuncSetAttribute(k_potrf, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
        PotrfArgs pa{}; pa.tile = d; pa.nt = nt; pa.in_smem = 1;
        for (int it = 0; it < 2; ++it) {
            cudaMemcpy(d, h.data(), nt * nt * 8, cudaMemcpyHostToDevice);
            k_potrf<<<1, kPotrfThreads, sm>>>(pa);
            cudaDeviceSynchronize();
        }
        long long t[4096];
        cudaMemcpyFromSymbol(t, g_potrf_trace, sizeof(t));
        int NB = ntp / 8;
        long long t0 = t[0];
        printf("nt=%d: per panel [gemm_start gemm_end chol_done trsm(K+1)_done] rel cycles\n", nt);
        for (int K = 0; K < NB; ++K) printf("  K=%2d %7lld %7lld %7lld %7lld | next-owner: gemm_done %7lld diag_seen %7lld solved %7lld\n", K, t[4*K]-t0, t[4*K+1]-t0, t[4*K+2]-t0, (K+1<NB)? t[4*K+3]-t0 : 0,
            (K+1<NB)? t[1000+4*K]-t0:0, (K+1<NB)? t[1000+4*K+1]-t0:0, (K+1<NB)? t[1000+4*K+2]-t0:0);
    }
}
