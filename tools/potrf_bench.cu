// Standalone POTRF latency + correctness (one CTA, k_potrf direct mode).
#include <cmath>
#include <cstdlib>
#include <cstdio>
#include <vector>
#include "../paper_2501_02483_b200/csrc/tc_kernels.cuh"
using namespace tc;
__global__ void k_potrf_many(PotrfArgs a, int nt) {
    extern __shared__ __align__(16) double smem[];
    a.tile += (size_t)blockIdx.x * nt * nt;
    potrf_task(a, smem);
}
int main(int argc, char** argv) {
    if (argc > 1) {  // profiling mode: 148 independent tiles, one CTA each
        const int nt = atoi(argv[1]), G = 148;
        std::vector<double> h((size_t)G * nt * nt);
        for (int b = 0; b < G; ++b)
            for (int j = 0; j < nt; ++j)
                for (int i = 0; i < nt; ++i) h[(size_t)b * nt * nt + j * nt + i] = (i == j) ? nt + 1.0 : 1.0 / (1 + i + j);
        double* d;
        cudaMalloc(&d, h.size() * 8);
        int ntp = (nt + 7) & ~7;
        size_t sm = potrf_smem_bytes(ntp, true);
        cudaFuncSetAttribute(k_potrf_many, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
        PotrfArgs pa{};
        pa.tile = d;
        pa.nt = nt;
        pa.in_smem = 1;
        for (int it = 0; it < 3; ++it) {
            cudaMemcpy(d, h.data(), h.size() * 8, cudaMemcpyHostToDevice);
            k_potrf_many<<<G, kPotrfThreads, sm>>>(pa, nt);
        }
        cudaDeviceSynchronize();
        printf("many: %s\n", cudaGetErrorString(cudaGetLastError()));
        return 0;
    }
    int* prog;
    cudaMalloc(&prog, 4);
    for (int pubmode = 0; pubmode < 2; ++pubmode)
    for (int nt : {8, 40, 64, 96, 120, 128, 160, 184}) {
        std::vector<double> h(nt * nt), out(nt * nt);
        for (int j = 0; j < nt; ++j)
            for (int i = 0; i < nt; ++i) h[j * nt + i] = (i == j) ? nt + 1.0 : 1.0 / (1 + i + j);
        double* d;
        int* info;
        cudaMalloc(&d, nt * nt * 8);
        cudaMalloc(&info, 4);
        int ntp = (nt + 7) & ~7;
        size_t sm = potrf_smem_bytes(ntp, true);
        cudaFuncSetAttribute(k_potrf, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
        PotrfArgs pa{};
        pa.tile = d;
        pa.nt = nt;
        pa.in_smem = 1;
        pa.info_out = info;
        if (pubmode) pa.prog = prog;
        float best = 1e9;
        for (int it = 0; it < 20; ++it) {
            cudaMemcpy(d, h.data(), nt * nt * 8, cudaMemcpyHostToDevice);
            cudaMemset(prog, 0, 4);
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
        int hinfo;
        cudaMemcpy(&hinfo, info, 4, cudaMemcpyDeviceToHost);
        cudaMemcpy(out.data(), d, nt * nt * 8, cudaMemcpyDeviceToHost);
        // residual |L L^T - A|
        double err = 0, nrm = 0;
        int bi = -1, bj = -1;
        for (int j = 0; j < nt; ++j)
            for (int i = j; i < nt; ++i) {
                double s = 0;
                for (int k = 0; k <= j; ++k) s += out[k * nt + i] * out[k * nt + j];
                if (fabs(s - h[j * nt + i]) > 1e-12 && bi < 0) { bi = i; bj = j; }
                err = fmax(err, fabs(s - h[j * nt + i]));
                nrm = fmax(nrm, fabs(h[j * nt + i]));
            }
        if (bi >= 0) printf("   first bad (row %d, col %d)\n", bi, bj);
        double up = 0;
        for (int j = 0; j < nt; ++j)
            for (int i = 0; i < j; ++i) up = fmax(up, fabs(out[j * nt + i]));
        printf("pub=%d nt=%3d k_potrf best %7.2f us  info %d  rel resid %.2e  upper %.1e  %s\n", pubmode, nt, best * 1e3, hinfo,
               err / nrm, up, cudaGetErrorString(cudaGetLastError()));
        cudaFree(d);
        cudaFree(info);
    }
}
