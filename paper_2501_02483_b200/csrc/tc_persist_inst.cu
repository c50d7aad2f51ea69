// Explicit instantiation of one group of k_persist variants (compiled once
// per group with -DTC_INST_GROUP=g so the heavy kernels build in parallel).
#define TC_PERSIST_ONLY 1
#include "tc_kernels.cuh"
#include "tc_persist_list.h"
namespace tc {
#define TC_INST(G, BM, BN, WGM, WGN, KS, MINB, SB) \
    TC_INST_##G(BM, BN, WGM, WGN, KS, MINB, SB)
#define TC_DO(BM, BN, WGM, WGN, KS, MINB, SB) template __global__ void k_persist<BM, BN, WGM, WGN, KS, MINB, SB>(const __grid_constant__ PersistArgs);
#define TC_SKIP(BM, BN, WGM, WGN, KS, MINB, SB)
#if TC_INST_GROUP == 0
#define TC_INST_0 TC_DO
#else
#define TC_INST_0 TC_SKIP
#endif
#if TC_INST_GROUP == 1
#define TC_INST_1 TC_DO
#else
#define TC_INST_1 TC_SKIP
#endif
#if TC_INST_GROUP == 2
#define TC_INST_2 TC_DO
#else
#define TC_INST_2 TC_SKIP
#endif
#if TC_INST_GROUP == 3
#define TC_INST_3 TC_DO
#else
#define TC_INST_3 TC_SKIP
#endif
#if TC_INST_GROUP == 4
#define TC_INST_4 TC_DO
#else
#define TC_INST_4 TC_SKIP
#endif
#if TC_INST_GROUP == 5
#define TC_INST_5 TC_DO
#else
#define TC_INST_5 TC_SKIP
#endif
#if TC_INST_GROUP == 6
#define TC_INST_6 TC_DO
#else
#define TC_INST_6 TC_SKIP
#endif
#if TC_INST_GROUP == 7
#define TC_INST_7 TC_DO
#else
#define TC_INST_7 TC_SKIP
#endif
TC_PERSIST_VARIANTS(TC_INST)
}  // namespace tc
