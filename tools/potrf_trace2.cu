#define TC_POTRF_TRACE 1
#include <cstdio>
#include <vector>
#include "../paper_2501_02483_b200/csrc/tc_kernels.cuh"
using namespace tc;
int main() {
    for (int nt : {120}) {
        std::vector<double> h(nt * nt);
        for (int j = 0; j < nt; ++j) for (int i = 0; i < nt; ++i) h[j * nt + i] = (i == j) ? nt + 1.0 : 1.0 / (1 + i + j);
        double* d; cudaMalloc(&d, nt * nt * 8);
        int ntp = (nt + 7) & ~7; size_t sm = potrf_smem_bytes(ntp, true);
        cudaFuncSetAttribute(k_potrf, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
        PotrfArgs pa{}; pa.tile = d; pa.nt = nt; pa.in_smem = 1;
        for (int it = 0; it < 3; ++it) {
            cudaMemcpy(d, h.data(), nt * nt * 8, cudaMemcpyHostToDevice);
            k_potrf<<<1, kPotrfThreads, sm>>>(pa);
            cudaDeviceSynchronize();
        }
        long long t[4096];
        cudaMemcpyFromSymbol(t, g_potrf_trace, sizeof(t));
        int NB = ntp / 8;
        long long t0 = t[3];
        printf("nt=%d rel cycles: diag[ready solve rank8 chol8 publish]  worker-of-K+1[gemm_last partial solve]\n", nt);
        for (int K = 0; K < NB; ++K) {
            printf("K=%2d", K);
            for (int x = 0; x < 8; ++x) printf(" %7lld", t[8 * K + x] ? t[8 * K + x] - t0 : -1);
            printf("\n");
        }
        for (int st = 0; st < 6; ++st) {
            printf("worker %d: [step1 step3 gotdiag step4]\n", st);
            for (int K = 0; K < NB; ++K) {
                long long* u = t + 512 + (st * 32 + K) * 4;
                if (!u[0] && !u[3]) continue;
                printf("  K=%2d %7lld %7lld %7lld %7lld\n", K, u[0] - t0, u[1] - t0, u[2] ? u[2] - t0 : -1, u[3] - t0);
            }
        }
    }
}
