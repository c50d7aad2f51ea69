// Standalone tile POTRF latency: packed shared-memory chain (in_smem = 1) vs
// the two-level path (L00 | L10 by DMMA | A11 -= L10 L10^T | L11), one CTA,
// k_potrf direct mode; residual |L L^T - A| / |A| checked on the host.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -I include -o tools/potrf_ab tools/potrf_ab.cu -lcuda
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <vector>
#include "../paper_2501_02483_b200/csrc/tc_kernels.cuh"
using namespace tc;
int main() {
    for (int nt : {64, 96, 120, 128, 160, 184, 192, 240, 256}) {
        for (int mode = 0; mode < 2; ++mode) {
            const int ntp = (nt + 7) & ~7;
            const bool packed = mode == 0;
            if (packed && potrf_packed_doubles(ntp) * 8 + ntp * 8 > 218 * 1024) continue;
            std::vector<double> h((size_t)nt * nt), out((size_t)nt * nt);
            for (int j = 0; j < nt; ++j)
                for (int i = 0; i < nt; ++i) h[j * nt + i] = (i == j) ? nt + 1.0 : 1.0 / (1 + i + j);
            double* d;
            int* info;
            cudaMalloc(&d, (size_t)nt * nt * 8);
            cudaMalloc(&info, 4);
            const size_t sm = potrf_smem_bytes(ntp, packed);
            cudaFuncSetAttribute(k_potrf, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
            PotrfArgs pa{};
            pa.tile = d;
            pa.nt = nt;
            pa.in_smem = packed;
            pa.info_out = info;
            float best = 1e9;
            for (int it = 0; it < 20; ++it) {
                cudaMemcpy(d, h.data(), (size_t)nt * nt * 8, cudaMemcpyHostToDevice);
                cudaEvent_t e0, e1;
                cudaEventCreate(&e0);
                cudaEventCreate(&e1);
                cudaEventRecord(e0);
                k_potrf<<<1, kPotrfThreads, sm>>>(pa);
                cudaEventRecord(e1);
                cudaEventSynchronize(e1);
                float ms;
                cudaEventElapsedTime(&ms, e0, e1);
                if (ms < best) best = ms;
            }
            int hinfo = -7;
            cudaMemcpy(&hinfo, info, 4, cudaMemcpyDeviceToHost);
            cudaMemcpy(out.data(), d, (size_t)nt * nt * 8, cudaMemcpyDeviceToHost);
            double err = 0, nrm = 0;
            for (int j = 0; j < nt; ++j)
                for (int i = j; i < nt; ++i) {
                    double s = 0;
                    for (int k = 0; k <= j; ++k) s += out[k * nt + i] * out[k * nt + j];
                    err += (s - h[j * nt + i]) * (s - h[j * nt + i]);
                    nrm += h[j * nt + i] * h[j * nt + i];
                }
            printf("nt %3d %-9s %8.2f us  info %d  rel resid %.2e  (%s)\n", nt, packed ? "packed" : "two-level", best * 1e3,
                   hinfo, sqrt(err / nrm), cudaGetErrorString(cudaGetLastError()));
            cudaFree(d);
            cudaFree(info);
        }
    }
    return 0;
}
