// Throughput of the gathered tile-update kernel in isolation.
#include <cstdio>
#include <vector>
#include <random>
#include "../paper_2501_02483_b200/csrc/tc_kernels.cuh"
using namespace tc;

template <int BM, int BN, int WGM, int WGN, int KS>
void run(int nt, int ncta_per_sm, int pairs, const char* name, int force_smem = 0) {
    using C = UpdCfg<BM, BN, WGM, WGN, KS>;
    int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    const int nitems = sms * ncta_per_sm;
    const int S = 64 + nitems;  // 64 operand tiles + one target per item (tile-blocks)
    double* st; cudaMalloc(&st, (size_t)S * nt * nt * 8);
    std::vector<double> h((size_t)S * nt * nt);
    std::mt19937_64 rng(1); std::uniform_real_distribution<double> U(-1, 1);
    for (auto& v : h) v = U(rng);
    cudaMemcpy(st, h.data(), h.size() * 8, cudaMemcpyHostToDevice);
    std::vector<Item> items; std::vector<Pair> pr;
    const int nrb = (nt + BM - 1) / BM, ncb = (nt + BN - 1) / BN;
    for (int i = 0; i < nitems; ++i) {
        const int blk = i % (nrb * ncb);
        Item it{64 + i, (blk % nrb) * BM, (blk / nrb) * BN, (int)pr.size(), 0, MODE_SUB};
        for (int p = 0; p < pairs; ++p) pr.push_back(Pair{(i * 7 + p * 3) % 64, (i * 5 + p * 11 + 1) % 64});
        it.p1 = (int)pr.size();
        items.push_back(it);
    }
    Item* di; Pair* dp;
    cudaMalloc(&di, items.size() * sizeof(Item)); cudaMalloc(&dp, pr.size() * sizeof(Pair));
    cudaMemcpy(di, items.data(), items.size() * sizeof(Item), cudaMemcpyHostToDevice);
    cudaMemcpy(dp, pr.data(), pr.size() * sizeof(Pair), cudaMemcpyHostToDevice);
    const int smem = force_smem > C::SMEM ? force_smem : C::SMEM;
    cudaFuncSetAttribute(k_update<BM, BN, WGM, WGN, KS>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    UpdArgs a{}; a.items = di; a.pairs = dp; a.storage = st; a.S = S; a.nt = nt;
    float best = 1e9;
    for (int r = 0; r < 5; ++r) {
        cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
        cudaEventRecord(e0);
        k_update<BM, BN, WGM, WGN, KS><<<nitems, C::NTH, smem>>>(a);
        cudaEventRecord(e1); cudaEventSynchronize(e1);
        float ms; cudaEventElapsedTime(&ms, e0, e1); if (ms < best) best = ms;
    }
    const double fl = 2.0 * BM * BN * (double)nt * pairs * nitems;
    int occ = 0; cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, k_update<BM, BN, WGM, WGN, KS>, C::NTH, smem);
    printf("%-22s nt=%3d ctas=%4d pairs=%2d occ/SM=%d  %.3f ms  %.2f TF/s  (err %s)\n", name, nt, nitems, pairs, occ, best,
           fl / (best * 1e-3) / 1e12, cudaGetErrorString(cudaGetLastError()));
    cudaFree(st); cudaFree(di); cudaFree(dp);
}

int main() {
    const int ONE = 150 * 1024;
    for (int pairs : {4, 16}) {
        run<64, 64, 2, 2, 2>(128, 1, pairs, "64x64 ks2 256t occ1", ONE);
        run<64, 64, 2, 2, 2>(128, 2, pairs, "64x64 ks2 256t");
        run<64, 64, 2, 2, 1>(128, 1, pairs, "64x64 ks1 128t occ1", ONE);
        run<64, 64, 2, 2, 1>(128, 3, pairs, "64x64 ks1 128t");
        run<80, 48, 2, 2, 2>(240, 1, pairs, "80x48 ks2 256t occ1", ONE);
        run<40, 40, 1, 1, 8>(120, 1, pairs, "40x40 ks8 256t occ1", ONE);
        run<40, 40, 1, 1, 4>(120, 1, pairs, "40x40 ks4 128t occ1", ONE);
        run<40, 40, 1, 1, 4>(120, 3, pairs, "40x40 ks4 128t");
        run<64, 64, 2, 2, 2>(192, 1, pairs, "64x64 ks2 256t occ1", ONE);
        run<64, 64, 2, 2, 2>(256, 1, pairs, "64x64 ks2 256t occ1", ONE);
    }
}
