// Phase timing of one gathered-update item (single pair, 40x40 block, K = nt) in one CTA.
#define TC_UPD_TRACE 1
#include <cstdio>
#include <vector>
#include "../paper_2501_02483_b200/csrc/tc_kernels.cuh"
using namespace tc;
template <int BM, int BN, int WGM, int WGN, int KS>
void run(int nt, const char* name) {
    using C = UpdCfg<BM, BN, WGM, WGN, KS>;
    std::vector<double> h(3 * nt * nt);
    for (size_t i = 0; i < h.size(); ++i) h[i] = 1.0 / (1 + i % 97);
    double* d;
    cudaMalloc(&d, h.size() * 8);
    cudaMemcpy(d, h.data(), h.size() * 8, cudaMemcpyHostToDevice);
    cudaFuncSetAttribute(k_update<BM, BN, WGM, WGN, KS>, cudaFuncAttributeMaxDynamicSharedMemorySize, C::SMEM);
    UpdArgs ua{};
    ua.storage = d;
    ua.S = 3;
    ua.nt = nt;
    ua.s_dst = 2;
    ua.s_a = 0;
    ua.s_b = 1;
    ua.s_mode = MODE_SUB;
    for (int it = 0; it < 3; ++it) {
        k_update<BM, BN, WGM, WGN, KS><<<1, C::NTH, C::SMEM>>>(ua);
        cudaDeviceSynchronize();
    }
    long long t[64];
    cudaMemcpyFromSymbol(t, g_upd_trace, sizeof(t));
    printf("%s nt=%d: prologue %lld, pairs %lld, stages:", name, nt, t[1] - t[0], t[2] - t[1]);
    for (int i = 0; i < 8 && t[3 + i] > t[2]; ++i) printf(" %lld", t[3 + i] - t[0]);
    printf(" | mainloop end %lld, reduce+stage %lld, rmw %lld, total %lld  (%s)\n", t[20] - t[0], t[21] - t[20],
           t[22] - t[21], t[22] - t[0], cudaGetErrorString(cudaGetLastError()));
}
int main() {
    run<40, 40, 1, 1, 8>(120, "persist40x40ks8");
    run<40, 40, 1, 1, 4>(120, "direct40x40ks4");
    run<64, 64, 2, 2, 2>(128, "persist64x64ks2");
    run<128, 64, 4, 2, 1>(128, "persist128x64");
    run<128, 128, 2, 4, 1>(128, "persist128x128");
}
