// tc_device.cu — C ABI of the device path: single-tile kernels, the
// run_ops / replay_residual plugin entries and the optimised launch plan.
// See include/tilechol_b200.h for the contract of every entry point.
#include <algorithm>
#include <cstdarg>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <memory>
#include <string>
#include <type_traits>
#include <vector>

#include "tc_kernels.cuh"
#include "tc_persist_list.h"
#include "tilechol_b200.h"

// k_persist variants are instantiated in tc_persist_inst.cu (parallel build)
namespace tc {
#define TC_EXTERN(G, BM, BN, WGM, WGN, KS, MINB, SB) \
    extern template __global__ void k_persist<BM, BN, WGM, WGN, KS, MINB, SB>(const __grid_constant__ PersistArgs);
TC_PERSIST_VARIANTS(TC_EXTERN)
#undef TC_EXTERN
}  // namespace tc

using namespace tc;

// ---------------------------------------------------------------- errors --
static thread_local std::string g_err;

static int set_err(int code, const char* fmt, ...) {
    char buf[512];
    va_list ap;
    va_start(ap, fmt);
    vsnprintf(buf, sizeof buf, fmt, ap);
    va_end(ap);
    g_err = buf;
    return code;
}

#define CK(call)                                                                          \
    do {                                                                                  \
        cudaError_t e_ = (call);                                                          \
        if (e_ != cudaSuccess)                                                            \
            return set_err(TC_ERR_CUDA, "%s:%d %s: %s", __FILE__, __LINE__, #call,       \
                           cudaGetErrorString(e_));                                       \
    } while (0)

extern "C" const char* tc_last_error(void) { return g_err.c_str(); }
extern "C" int32_t tc_abi_version(void) { return 1; }
extern "C" int32_t tc_device_count(void) {
    int n = 0;
    if (cudaGetDeviceCount(&n) != cudaSuccess) {
        cudaGetLastError();
        return 0;
    }
    return n;
}

// ----------------------------------------------------- kernel selection --
namespace {

struct UpdKernel {
    void (*fn)(UpdArgs);
    int BM, BN, nth, smem;
};

template <int BM, int BN, int WGM, int WGN, int KS>
UpdKernel mk_upd() {
    using C = UpdCfg<BM, BN, WGM, WGN, KS>;
    return UpdKernel{k_update<BM, BN, WGM, WGN, KS>, BM, BN, C::NTH, C::SMEM};
}

// Block shape per tile size: blocks that divide nt exactly where possible so
// no MMA work is wasted on padding (120 -> 40x40, 160/320 -> 80x40,
// 240/480 -> 80x48), small / odd sizes fall back to predicated 32x32.
// Large blocks for nt % 128 == 0: 128x64 half tiles (4x2 warps of 32x32, no
// split-K) or whole 128x128 tiles; TC_UPD_SHAPE=128x64 / 128x128 / 64x64.
int big_shape(int nt) {
    if (nt % 128 != 0) return 0;
    const char* f = getenv("TC_UPD_SHAPE");
    if (f && !strcmp(f, "128x64")) return 1;
    if (f && !strcmp(f, "128x128")) return 2;
    return 0;
}
UpdKernel pick_upd(int nt) {
    switch (big_shape(nt)) {
        case 1: return mk_upd<128, 64, 4, 2, 1>();
        case 2: return mk_upd<128, 128, 2, 4, 1>();
        default: break;
    }
    if (const char* f = getenv("TC_PERSIST_SHAPE")) {  // tuning override (kept in step with pick_persist)
        if (!strcmp(f, "64")) return mk_upd<64, 64, 2, 2, 1>();
        if (!strcmp(f, "32")) return mk_upd<32, 32, 2, 2, 1>();
        if (!strcmp(f, "40")) return mk_upd<40, 40, 1, 1, 4>();
    }
    if (nt % 64 == 0) return mk_upd<64, 64, 2, 2, 1>();
    if (nt % 80 == 0 && nt % 48 == 0) return mk_upd<80, 48, 2, 2, 1>();
    if (nt % 80 == 0) return mk_upd<80, 40, 2, 1, 2>();
    if (nt % 40 == 0) return mk_upd<40, 40, 1, 1, 4>();
    if (nt >= 96) return mk_upd<64, 64, 2, 2, 1>();
    return mk_upd<32, 32, 2, 2, 1>();
}

// Small square blocks for the one-pair L(k) items on the critical path: a
// 40x40x120 block costs ~7 us on one SM (8-way split-K tree epilogue
// included); 24x24 spreads the same GEMM over ~3x more SMs at ~1/3 the
// per-CTA work.  0 = none (tile size not a multiple of 24 or 32).
int small_block(int nt) {
    if (getenv("TC_NO_SMALL_LAST")) return 0;
    if (nt % 24 == 0 && nt >= 96) return 24;
    if (nt % 32 == 0 && nt >= 96) return 32;
    return 0;
}
UpdKernel pick_upd_small(int nt) {
    switch (small_block(nt)) {
        case 24: return mk_upd<24, 24, 1, 1, 4>();
        case 32: return mk_upd<32, 32, 1, 1, 4>();
        default: return UpdKernel{};
    }
}

struct PersistKernel {
    void (*fn)(PersistArgs);
    int BM, BN, smem;
    int lda, ldb, kc;  // update operand staging: padded column strides, k-chunk (TMA boxes)
};

template <int BM, int BN, int WGM, int WGN, int KS, int SB>
PersistKernel mk_persist_sb(int minb) {
    using U = UpdCfg<BM, BN, WGM, WGN, KS>;
    return PersistKernel{minb == 2 ? k_persist<BM, BN, WGM, WGN, KS, 2, SB> : k_persist<BM, BN, WGM, WGN, KS, 1, SB>,
                         BM, BN, U::SMEM, U::LDA, U::LDB, U::KC};
}
// Only the small-block variants a shape can meet are instantiated (compile
// time): small_block(nt) for the tile sizes that select each update shape.
template <int BM, int BN, int WGM, int WGN, int KS, int... SBS>
PersistKernel mk_persist(int minb, int nt) {
    const int sb = small_block(nt);
    PersistKernel out{};
    auto try_one = [&](auto tag) {
        constexpr int SB = decltype(tag)::value;
        if (sb == SB) out = mk_persist_sb<BM, BN, WGM, WGN, KS, SB>(minb);
    };
    (try_one(std::integral_constant<int, SBS>{}), ...);
    return out;  // fn == nullptr: no variant for this tile size (plan creation fails loudly)
}

// same block shapes as pick_upd, 256-thread variants (KSPLIT doubled);
// minb = minimum resident CTAs per SM the variant is compiled for
template <int BM, int BN, int WGM, int WGN, int KS, int SB>
PersistKernel mk_persist1() {
    using U = UpdCfg<BM, BN, WGM, WGN, KS>;
    return PersistKernel{k_persist<BM, BN, WGM, WGN, KS, 1, SB>, BM, BN, U::SMEM, U::LDA, U::LDB, U::KC};
}
PersistKernel pick_persist(int nt, int minb) {
    if (small_block(nt) == 32) {
        switch (big_shape(nt)) {
            case 1: return mk_persist1<128, 64, 4, 2, 1, 32>();
            case 2: return mk_persist1<128, 128, 2, 4, 1, 32>();
            default: break;
        }
    }
    if (nt % 64 == 0) return mk_persist<64, 64, 2, 2, 2, 0, 24, 32>(minb, nt);
    if (nt % 80 == 0 && nt % 48 == 0) return mk_persist<80, 48, 2, 2, 2, 24>(minb, nt);
    if (nt % 80 == 0) return mk_persist<80, 40, 2, 1, 4, 0, 32>(minb, nt);
    if (nt % 40 == 0) return mk_persist<40, 40, 1, 1, 8, 0, 24>(minb, nt);
    if (nt >= 96) return mk_persist<64, 64, 2, 2, 2, 0, 24, 32>(minb, nt);
    return mk_persist<32, 32, 2, 2, 2, 0>(minb, nt);
}

int prep_kernel(const void* fn, int smem) {
    // always opt in: static shared memory plus a dynamic size just below 48 KB
    // can exceed the default 48 KB window
    CK(cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
    return TC_OK;
}

// packed lower block rows in shared memory up to ntp = 184, else in place
// smallest tile size factored by the two-level POTRF (TC_POTRF2_MIN; default:
// only tiles whose packed triangle does not fit shared memory)
int potrf2_min() {
    static const int v = getenv("TC_POTRF2_MIN") ? atoi(getenv("TC_POTRF2_MIN")) : 185;
    return v;
}

size_t potrf_smem(int nt, bool* in_smem) {
    const int ntp = (nt + 7) & ~7;
    const size_t packed = potrf_packed_doubles(ntp) * 8 + (size_t)ntp * 8;
    if (nt % 8 == 0 && nt >= 16 && nt <= 256 && nt >= potrf2_min()) {
        *in_smem = false;
        return potrf_smem_bytes(ntp, false);
    }
    if (packed <= 218 * 1024) {
        *in_smem = true;
        return packed;
    }
    *in_smem = false;
    return potrf_smem_bytes(ntp, false);  // two-level path (nt <= 256) or 1/diag only
}

bool potrf_supported(int nt) {
    bool in_smem;
    potrf_smem(nt, &in_smem);
    return in_smem || (nt % 8 == 0 && nt <= 768);  // in place: 8-row blocks, <= 96 of them
}

constexpr int kMaxTrsmNt = 1024;

// direct TRSM kernel for a tile size: 32-row strips, 16-row strips when the
// 32-row X strip plus two staging buffers would not fit shared memory
struct TrsmK {
    void (*fn)(TrsmArgs);
    int rows;
    size_t smem;
};
TrsmK trsm_direct(int nt) {
    if (trsm_fits<32>(nt, 225 * 1024)) return TrsmK{k_trsm<32>, 32, trsm_smem_bytes<32>(nt)};
    return TrsmK{k_trsm<16>, 16, trsm_smem_bytes<16>(nt)};
}
size_t trsm_smem_rows(int rows, int nt) {
    return rows == 64 ? trsm_smem_bytes<64>(nt) : rows == 32 ? trsm_smem_bytes<32>(nt) : trsm_smem_bytes<16>(nt);
}
size_t trsm_ring_rows(int rows, int nt, int nb) {
    return rows == 64 ? trsm_smem_ring<64>(nt, nb) : rows == 32 ? trsm_smem_ring<32>(nt, nb) : trsm_smem_ring<16>(nt, nb);
}

inline double* tptr(double* st, double* sc, int64_t S, int64_t s, int nt) {
    const size_t nt2 = (size_t)nt * nt;
    return s < S ? st + (size_t)s * nt2 : sc + (size_t)(s - S) * nt2;
}

int launch_update_single(const UpdKernel& K, double* st, double* sc, int64_t S, int nt, int64_t dst,
                         int64_t a, int64_t b, const int64_t* fail, cudaStream_t s) {
    int r = prep_kernel((const void*)K.fn, K.smem);
    if (r) return r;
    UpdArgs ua{};
    ua.storage = st;
    ua.scratch = sc;
    ua.S = S;
    ua.fail = fail;
    ua.nt = nt;
    ua.s_dst = (int32_t)dst;
    ua.s_a = (int32_t)a;
    ua.s_b = (int32_t)b;
    ua.s_mode = MODE_SUB;
    const int nrb = (nt + K.BM - 1) / K.BM, ncb = (nt + K.BN - 1) / K.BN;
    K.fn<<<nrb * ncb, K.nth, K.smem, s>>>(ua);
    CK(cudaGetLastError());
    return TC_OK;
}

int launch_potrf_direct(double* tile, int nt, int32_t* info_dev, const int64_t* fail, int64_t op_index,
                        int64_t* fail_p, int32_t* fail_info, cudaStream_t s) {
    if (!potrf_supported(nt))
        return set_err(TC_ERR_ARG, "potrf: nt=%d > 160 must be a multiple of 8", nt);
    bool in_smem;
    const size_t sm = potrf_smem(nt, &in_smem);
    int r = prep_kernel((const void*)k_potrf, (int)sm);
    if (r) return r;
    PotrfArgs pa{};
    pa.tile = tile;
    pa.info_out = info_dev;
    pa.nt = nt;
    pa.in_smem = in_smem;
    pa.fail = fail;
    pa.op_index = op_index;
    pa.fail_p = fail_p;
    pa.fail_info = fail_info;
    k_potrf<<<1, kPotrfThreads, sm, s>>>(pa);
    CK(cudaGetLastError());
    return TC_OK;
}

int launch_trsm_direct(const double* L, double* X, int nt, int32_t* info_dev, const int64_t* fail, int64_t op_index,
                       int64_t* fail_p, int32_t* fail_info, cudaStream_t s) {
    if (nt > kMaxTrsmNt) return set_err(TC_ERR_ARG, "trsm: nt=%d > %d unsupported", nt, kMaxTrsmNt);
    const TrsmK TK = trsm_direct(nt);
    const size_t sm = TK.smem;
    int r = prep_kernel((const void*)TK.fn, (int)sm);
    if (r) return r;
    TrsmArgs ta{};
    ta.L = L;
    ta.X = X;
    ta.nt = nt;
    ta.fail = fail;
    ta.check_zero = 1;
    ta.info_out = info_dev;
    ta.op_index = op_index;
    ta.fail_p = fail_p;
    ta.fail_info = fail_info;
    dim3 grid((nt + TK.rows - 1) / TK.rows, 1);
    TK.fn<<<grid, 4 * TK.rows, sm, s>>>(ta);
    CK(cudaGetLastError());
    return TC_OK;
}

int elem_grid(int nt) {
    const size_t n2 = (size_t)nt * nt;
    return (int)std::min<size_t>((n2 + 255) / 256, 592);
}

// small device scratch for status words of synchronous entry points
struct StatusBuf {
    int64_t* fail_p = nullptr;
    int32_t* info = nullptr;
    int alloc(cudaStream_t s) {
        void* p = nullptr;
        CK(cudaMallocAsync(&p, 16, s));
        fail_p = (int64_t*)p;
        info = (int32_t*)((char*)p + 8);
        const int64_t init[2] = {kNoFail, (int64_t)-1};
        CK(cudaMemcpyAsync(p, init, 16, cudaMemcpyHostToDevice, s));
        return TC_OK;
    }
    void release(cudaStream_t s) {
        if (fail_p) cudaFreeAsync(fail_p, s);
        fail_p = nullptr;
    }
};

}  // namespace

// ------------------------------------------------------ tile entry points --
extern "C" int tc_potrf_tile(double* a, int32_t nt, void* stream, int32_t* info) {
    if (!a || nt < 1 || !info) return set_err(TC_ERR_ARG, "potrf_tile: bad arguments");
    cudaStream_t s = (cudaStream_t)stream;
    StatusBuf sb;
    int r = sb.alloc(s);
    if (r) return r;
    r = launch_potrf_direct(a, nt, sb.info, nullptr, 0, nullptr, nullptr, s);
    if (r) return r;
    CK(cudaMemcpyAsync(info, sb.info, 4, cudaMemcpyDeviceToHost, s));
    sb.release(s);
    CK(cudaStreamSynchronize(s));
    return TC_OK;
}

extern "C" int tc_trsm_tile(const double* l, double* x, int32_t nt, void* stream, int32_t* info) {
    if (!l || !x || nt < 1 || !info) return set_err(TC_ERR_ARG, "trsm_tile: bad arguments");
    cudaStream_t s = (cudaStream_t)stream;
    StatusBuf sb;
    int r = sb.alloc(s);
    if (r) return r;
    r = launch_trsm_direct(l, x, nt, sb.info, nullptr, 0, nullptr, nullptr, s);
    if (r) return r;
    CK(cudaMemcpyAsync(info, sb.info, 4, cudaMemcpyDeviceToHost, s));
    sb.release(s);
    CK(cudaStreamSynchronize(s));
    return TC_OK;
}

extern "C" int tc_syrk_tile(const double* a, double* c, int32_t nt, void* stream) {
    if (!a || !c || nt < 1) return set_err(TC_ERR_ARG, "syrk_tile: bad arguments");
    // two-slot view: slot 0 = c, slot 1 = a (via scratch pointer trick)
    const UpdKernel K = pick_upd(nt);
    return launch_update_single(K, c, const_cast<double*>(a), 1, nt, 0, 1, 1, nullptr, (cudaStream_t)stream);
}

extern "C" int tc_gemm_tile(const double* a, const double* b, double* c, int32_t nt, void* stream) {
    if (!a || !b || !c || nt < 1) return set_err(TC_ERR_ARG, "gemm_tile: bad arguments");
    // c -= b a^T : kernel computes C -= A B^T with A = b (slot 1), B = a (slot 2)
    // slots: 0 -> c (storage), >= 1 -> scratch; place b and a contiguously is not
    // possible in general, so run with storage = c and scratch = b when a == b,
    // else use two launches-free trick: pass a as storage base of a 3-slot view.
    const UpdKernel K = pick_upd(nt);
    cudaStream_t s = (cudaStream_t)stream;
    // Build a tiny device pointer table: the single-op mode addresses tiles as
    // storage + s*nt^2 / scratch + (s-S)*nt^2, so use S = 1 with storage = c
    // and scratch = b for A, and a separate launch cannot express B = a.
    // Instead compute with S large-offset arithmetic: pick base = min pointer.
    const double* ptrs[3] = {c, b, a};
    const double* base = std::min({ptrs[0], ptrs[1], ptrs[2]});
    const size_t nt2 = (size_t)nt * nt;
    auto off = [&](const double* p) -> int64_t {
        const ptrdiff_t d = p - base;
        return (d % (ptrdiff_t)nt2 == 0) ? (int64_t)(d / (ptrdiff_t)nt2) : -1;
    };
    const int64_t oc = off(c), ob = off(b), oa = off(a);
    if (oc >= 0 && ob >= 0 && oa >= 0 && std::max({oc, ob, oa}) < INT32_MAX) {
        return launch_update_single(K, const_cast<double*>(base), nullptr, INT64_MAX, nt, oc, ob, oa, nullptr, s);
    }
    // unaligned distinct allocations: stage a and b into one temporary buffer
    double* tmp = nullptr;
    CK(cudaMallocAsync((void**)&tmp, 2 * nt2 * 8, s));
    CK(cudaMemcpyAsync(tmp, b, nt2 * 8, cudaMemcpyDeviceToDevice, s));
    CK(cudaMemcpyAsync(tmp + nt2, a, nt2 * 8, cudaMemcpyDeviceToDevice, s));
    int r = launch_update_single(K, c, tmp, 1, nt, 0, 1, 2, nullptr, s);
    cudaFreeAsync(tmp, s);
    return r;
}

extern "C" int tc_geadd_tile(const double* t, double* c, int32_t nt, void* stream) {
    if (!t || !c || nt < 1) return set_err(TC_ERR_ARG, "geadd_tile: bad arguments");
    k_geadd<<<elem_grid(nt), 256, 0, (cudaStream_t)stream>>>(nullptr, c, const_cast<double*>(t), 1, 1, 0, nt, nullptr);
    CK(cudaGetLastError());
    return TC_OK;
}

// ----------------------------------------------------------- run_ops --
extern "C" int tc_run_ops(double* storage, int64_t S, double* scratch, int64_t R, int32_t nt,
                          const int8_t* op, const int64_t* dst, const int64_t* src1, const int64_t* src2,
                          int64_t n_ops, int64_t start, int64_t stop, void* stream, int64_t* out_p,
                          int32_t* out_info) {
    if (nt < 1 || S < 0 || R < 0 || start < 0 || stop > n_ops || start > stop || !out_p || !out_info)
        return set_err(TC_ERR_ARG, "run_ops: bad arguments");
    if (stop > start && (!op || !dst)) return set_err(TC_ERR_ARG, "run_ops: null op arrays");
    const int64_t lim = S + R;
    for (int64_t p = start; p < stop; ++p) {
        const int t = op[p];
        auto bad = [&](int64_t v) { return v < 0 || v >= lim; };
        if (bad(dst[p])) return set_err(TC_ERR_ARG, "run_ops: op %lld dst %lld out of range", (long long)p, (long long)dst[p]);
        if ((t == TC_GEMM || t == TC_SYRK || t == TC_TRSM || t == TC_GEADD) && (!src1 || bad(src1[p])))
            return set_err(TC_ERR_ARG, "run_ops: op %lld src1 out of range", (long long)p);
        if (t == TC_GEMM && (!src2 || bad(src2[p])))
            return set_err(TC_ERR_ARG, "run_ops: op %lld src2 out of range", (long long)p);
        if ((t == TC_POTRF && !potrf_supported(nt)) || (t == TC_TRSM && nt > kMaxTrsmNt))
            return set_err(TC_ERR_ARG, "run_ops: nt=%d unsupported for op %d", nt, t);
    }
    cudaStream_t s = (cudaStream_t)stream;
    StatusBuf sb;
    int r = sb.alloc(s);
    if (r) return r;
    const UpdKernel K = pick_upd(nt);
    for (int64_t p = start; p < stop && r == TC_OK; ++p) {
        const int t = op[p];
        double* d = tptr(storage, scratch, S, dst[p], nt);
        switch (t) {
            case TC_GEMM:
                r = launch_update_single(K, storage, scratch, S, nt, dst[p], src2[p], src1[p], sb.fail_p, s);
                break;
            case TC_SYRK:
                r = launch_update_single(K, storage, scratch, S, nt, dst[p], src1[p], src1[p], sb.fail_p, s);
                break;
            case TC_TRSM:
                r = launch_trsm_direct(tptr(storage, scratch, S, src1[p], nt), d, nt, nullptr, sb.fail_p, p,
                                       sb.fail_p, sb.info, s);
                break;
            case TC_POTRF:
                r = launch_potrf_direct(d, nt, nullptr, sb.fail_p, p, sb.fail_p, sb.info, s);
                break;
            case TC_GEADD:
                k_geadd<<<elem_grid(nt), 256, 0, s>>>(nullptr, storage, scratch, S, src1[p], dst[p], nt, sb.fail_p);
                break;
            default:  // reference: any other code zeroes the target tile
                k_zero<<<elem_grid(nt), 256, 0, s>>>(storage, scratch, S, dst[p], nt, sb.fail_p);
                break;
        }
        if (r == TC_OK) {
            cudaError_t e = cudaGetLastError();
            if (e != cudaSuccess) r = set_err(TC_ERR_CUDA, "run_ops launch: %s", cudaGetErrorString(e));
        }
    }
    int64_t hp[2];
    if (r == TC_OK) {
        CK(cudaMemcpyAsync(hp, sb.fail_p, 16, cudaMemcpyDeviceToHost, s));
    }
    sb.release(s);
    CK(cudaStreamSynchronize(s));
    if (r) return r;
    if (hp[0] == kNoFail) {
        *out_p = stop;
        *out_info = -1;
    } else {
        *out_p = hp[0];
        *out_info = (int32_t)(hp[1] & 0xffffffff);
    }
    return TC_OK;
}

// --------------------------------------------------- replay_residual --
namespace {
void tile_blocks(int nt, int BM, int BN, bool lower_only, std::vector<std::pair<int, int>>& out) {
    out.clear();
    for (int c0 = 0; c0 < nt; c0 += BN)
        for (int r0 = 0; r0 < nt; r0 += BM) {
            if (lower_only && r0 + BM - 1 < c0) continue;
            out.emplace_back(r0, c0);
        }
}

template <class T>
int upload(const std::vector<T>& v, T** d, cudaStream_t s) {
    *d = nullptr;
    if (v.empty()) return TC_OK;
    CK(cudaMallocAsync((void**)d, v.size() * sizeof(T), s));
    CK(cudaMemcpyAsync(*d, v.data(), v.size() * sizeof(T), cudaMemcpyHostToDevice, s));
    return TC_OK;
}
}  // namespace

extern "C" int tc_replay_residual(const double* storage, const double* tmpl, int64_t S, int32_t nt,
                                  const int8_t* op, const int64_t* dst, const int64_t* src1,
                                  const int64_t* src2, int64_t n_ops, const uint8_t* diag_slot, void* stream,
                                  double* out_err2) {
    if (nt < 1 || S < 1 || !out_err2 || !diag_slot || (n_ops > 0 && (!op || !dst)))
        return set_err(TC_ERR_ARG, "replay_residual: bad arguments");
    const UpdKernel K = pick_upd(nt);
    std::vector<Item> items;
    std::vector<Pair> pairs;
    std::vector<std::pair<int, int>> blocks;
    tile_blocks(nt, K.BM, K.BN, false, blocks);
    for (int64_t p = 0; p < n_ops;) {
        const int64_t d = dst[p];
        if (d < 0 || d >= S) return set_err(TC_ERR_ARG, "replay_residual: dst out of range (scratch not allowed)");
        const int32_t p0 = (int32_t)pairs.size();
        int64_t q = p;
        for (; q < n_ops && dst[q] == d; ++q) {
            int64_t a, b;
            switch (op[q]) {
                case TC_POTRF: a = d; b = d; break;
                case TC_SYRK: a = src1[q]; b = src1[q]; break;
                case TC_TRSM: a = d; b = src1[q]; break;
                default: a = src2[q]; b = src1[q]; break;
            }
            if (a < 0 || a >= S || b < 0 || b >= S) return set_err(TC_ERR_ARG, "replay_residual: source out of range");
            pairs.push_back(Pair{(int32_t)a, (int32_t)b});
        }
        const int32_t p1 = (int32_t)pairs.size();
        for (auto& bl : blocks) items.push_back(Item{(int32_t)d, bl.first, bl.second, p0, p1, MODE_RESID});
        p = q;
    }
    cudaStream_t s = (cudaStream_t)stream;
    if (items.empty()) {
        *out_err2 = 0.0;
        return TC_OK;
    }
    Item* di = nullptr;
    Pair* dp = nullptr;
    uint8_t* dd = nullptr;
    double* part = nullptr;
    int r = upload(items, &di, s);
    if (!r) r = upload(pairs, &dp, s);
    std::vector<uint8_t> dg(diag_slot, diag_slot + S);
    if (!r) r = upload(dg, &dd, s);
    if (!r) {
        CK(cudaMallocAsync((void**)&part, (items.size() + 1) * 8, s));
        r = prep_kernel((const void*)K.fn, K.smem);
    }
    if (!r) {
        const int64_t chunk = 1 << 30;
        for (int64_t base = 0; base < (int64_t)items.size() && !r; base += chunk) {
            UpdArgs ua{};
            ua.items = di;
            ua.pairs = dp;
            ua.storage = const_cast<double*>(storage);
            ua.S = S;
            ua.nt = nt;
            ua.item_base = (int32_t)base;
            ua.tmpl = tmpl;
            ua.diag = dd;
            ua.resid_out = part;
            const int64_t cnt = std::min<int64_t>(chunk, (int64_t)items.size() - base);
            K.fn<<<(unsigned)cnt, K.nth, K.smem, s>>>(ua);
            cudaError_t e = cudaGetLastError();
            if (e != cudaSuccess) r = set_err(TC_ERR_CUDA, "replay launch: %s", cudaGetErrorString(e));
        }
        if (!r) {
            k_sum_fixed<<<1, 256, 0, s>>>(part, (int64_t)items.size(), 1.0, part + items.size());
            CK(cudaMemcpyAsync(out_err2, part + items.size(), 8, cudaMemcpyDeviceToHost, s));
        }
    }
    if (di) cudaFreeAsync(di, s);
    if (dp) cudaFreeAsync(dp, s);
    if (dd) cudaFreeAsync(dd, s);
    if (part) cudaFreeAsync(part, s);
    CK(cudaStreamSynchronize(s));
    return r;
}

// ======================================================================
// Optimised launch plan
// ======================================================================
namespace {

enum LaunchKind { L_UPD = 0, L_POTRF = 1, L_TRSM = 2, L_COMBINE = 3, L_LOGDET = 4 };

// trace classification of a launch (tc_plan_trace launch_meta bits 8..10)
constexpr int kTagChain = 1 << 8, kTagMid = 1 << 9, kTagSub = 1 << 10;
struct Launch {
    int kind = 0;
    int high = 0;                // critical-path priority
    int64_t off = 0, cnt = 0;    // items (UPD) / targets (TRSM)
    int32_t k = -1;              // column (POTRF/TRSM)
    int64_t slot = -1;           // POTRF slot / TRSM L slot / COMBINE target
    int64_t scratch0 = 0;        // COMBINE
    uint32_t live = 0;           // COMBINE
    int cls = 0;                 // profiling class: 0 bulk, 1 last, 2 potrf, 3 trsm, 4 combine, 5 logdet, 6 split-K chunk
    int small = 0;               // UPD items use the small latency block (L(k) launches)
    int tag = 0;                 // trace classification bits (kTag*)
    double flops = 0.0;          // algorithmic flops of this launch
    std::vector<int32_t> deps;
};

struct Lane {
    Ctx* d_ctx = nullptr;
    int64_t* d_fail = nullptr;
    double* d_ld = nullptr;      // [T + 1] partials + result
    double* d_scratch = nullptr;
    cudaGraphExec_t exec = nullptr;
    cudaGraph_t graph = nullptr;
    int32_t* d_pstate = nullptr;  // persistent: [remaining | deps_left | ticket]
    int32_t* d_prog = nullptr;    // persistent fused: per-column POTRF panel progress [T]
    int64_t* d_trace = nullptr;   // persistent: per-task timestamps (tc_plan_trace only)
    int32_t* d_xctr = nullptr;    // persistent: fused diagonal SYRK TRSM warp panel flags [T][32]
    Ctx h{};
};

}  // namespace

struct tc_plan {
    int64_t n = 0;
    int nt = 0;
    int T = 0;
    int64_t S = 0;
    tc_plan_opts opts{};
    int W = 0;
    std::vector<int32_t> frow, fcol;
    std::vector<int64_t> cs;            // column -> first slot
    std::vector<Launch> launches;
    std::vector<Item> items;
    std::vector<Pair> pairs;
    std::vector<int32_t> tgts;          // TRSM targets
    int64_t R = 0;                      // scratch tiles per lane
    double flops = 0.0;
    UpdKernel upd{};
    UpdKernel upd_small{};              // L(k): one-pair items in small blocks (latency), fn == null if none
    // device copies
    Item* d_items = nullptr;
    Pair* d_pairs = nullptr;
    int32_t* d_tgts = nullptr;
    int64_t* d_diag_slots = nullptr;
    // solve metadata: per column off-diagonal slots and rows
    std::vector<int64_t> sol_off;
    int32_t* d_sol_slots = nullptr;   // backward sweep: off-diagonal slots of column k, rows ascending
    int32_t* d_sol_rows = nullptr;
    int64_t* d_sol_off = nullptr;     // [T+1]
    int64_t* d_row_ptr = nullptr;     // forward sweep: off-diagonal tiles of row k, columns ascending
    int32_t* d_row_col = nullptr;
    int32_t* d_row_slot = nullptr;
    std::vector<Lane> lanes;
    int prio_hi = 0, prio_lo = 0;
    int dev = 0;
    // per-column launch ids (persistent ticket order)
    std::vector<int32_t> colB, colBd, colM, colMd, colL, colLc, colLo, colPot, colTrsm, colTrsmC;
    std::vector<std::vector<int32_t>> colComb, colChunk;
    // persistent executor
    std::vector<PTask> ptasks;
    std::vector<PLaunch> plaunch;
    std::vector<int32_t> p_remaining, p_deps, p_succ_ptr, p_succ;
    PTask* d_ptasks = nullptr;
    PLaunch* d_plaunch = nullptr;
    int32_t* d_p_init = nullptr;  // [remaining | deps_left] pristine copy
    int32_t* d_succ_ptr = nullptr;
    int32_t* d_succ = nullptr;
    size_t persist_smem = 0;
    bool fuse = true;  // persistent executor: TRSM(k) streams POTRF(k)'s panels
    int persist_trsm_ring = 0;  // 0 = auto staging, >0 = strip ring of that many buffers
    int persist_minb = 2;
    int persist_trsm_rows = 64;  // TRSM strip rows of the persistent executor
    PersistKernel pkern{};       // the persistent kernel variant chosen at plan time
    bool persist_tma = false;    // update operands through TMA tensor maps
    int persist_grid = 0;
    // fused diagonal SYRK: POTRF(k) applies the last update of its diagonal
    // tile itself, consuming L(k, n_last) panel by panel from TRSM(n_last)
    std::vector<int64_t> xslot_of_col;  // [T] slot of L(k, n_last) or -1
    int32_t* d_xctr_of_slot = nullptr;  // [S] consuming column or -1
    int nfused = 0;
};

namespace {

int64_t find_slot(const tc_plan& P, int32_t m, int32_t c) {
    // slots of column c are [cs[c], cs[c+1]) with ascending rows
    const int32_t* b = P.frow.data() + P.cs[c];
    const int32_t* e = P.frow.data() + P.cs[c + 1];
    const int32_t* it = std::lower_bound(b, e, m);
    return (it != e && *it == m) ? (int64_t)(it - P.frow.data()) : -1;
}

int build_persistent(tc_plan& P);

// TC_CRIT=0: one L_off(k) / TRSM(k) launch for every off-diagonal target
static bool crit_split() {
    static const bool v = !(getenv("TC_CRIT") && atoi(getenv("TC_CRIT")) == 0);
    return v;
}
// TC_BSPLIT=0: one bulk-update launch B(k) per column (diagonal tile included)
static bool b_split() {
    static const bool v = !(getenv("TC_BSPLIT") && atoi(getenv("TC_BSPLIT")) == 0);
    return v;
}
// TC_MSPLIT=0: one near-update launch M(k) per column (diagonal tile included)
static bool m_split() {
    static const bool v = !(getenv("TC_MSPLIT") && atoi(getenv("TC_MSPLIT")) == 0);
    return v;
}

int build_plan(tc_plan& P) {
    const int T = P.T, nt = P.nt;
    const int64_t S = P.S;
    // column starts, validation
    P.cs.assign(T + 1, 0);
    for (int64_t s = 0; s < S; ++s) {
        if (P.fcol[s] < 0 || P.fcol[s] >= T || P.frow[s] < P.fcol[s] || P.frow[s] >= T)
            return set_err(TC_ERR_ARG, "plan: slot %lld out of the lower tile triangle", (long long)s);
        if (s > 0 && (P.fcol[s] < P.fcol[s - 1] || (P.fcol[s] == P.fcol[s - 1] && P.frow[s] <= P.frow[s - 1])))
            return set_err(TC_ERR_ARG, "plan: slots not in (col,row) order");
        P.cs[P.fcol[s] + 1]++;
    }
    for (int k = 0; k < T; ++k) P.cs[k + 1] += P.cs[k];
    // lookahead < 0: automatic -- 3 on wide-column plans (>= 20 tiles per
    // column on average, e.g. C4 @128 with 22: 480 vs 507 ms at 4), 4
    // otherwise (C3 @128 with 18.8: 77 vs 87 ms at 3)
    if (P.opts.lookahead < 0) P.opts.lookahead = S >= 20 * (int64_t)T ? 3 : 4;
    for (int k = 0; k < T; ++k)
        if (P.cs[k + 1] == P.cs[k] || P.frow[P.cs[k]] != k)
            return set_err(TC_ERR_ARG, "plan: diagonal tile %d missing", k);
    // row lists (n ascending): L(k, n) slots
    std::vector<int64_t> rp(T + 1, 0);
    for (int64_t s = 0; s < S; ++s)
        if (P.frow[s] != P.fcol[s]) rp[P.frow[s] + 1]++;
    for (int k = 0; k < T; ++k) rp[k + 1] += rp[k];
    std::vector<int32_t> rn(rp[T]);
    std::vector<int64_t> rs(rp[T]);
    {
        std::vector<int64_t> fill(rp.begin(), rp.end() - 1);
        for (int64_t s = 0; s < S; ++s)
            if (P.frow[s] != P.fcol[s]) {
                const int64_t at = fill[P.frow[s]]++;
                rn[at] = P.fcol[s];
                rs[at] = s;
            }
    }
    std::vector<int32_t> parent(T, -1);
    for (int c = 0; c < T; ++c)
        if (P.cs[c + 1] - P.cs[c] > 1) parent[c] = P.frow[P.cs[c] + 1];

    // ---- pass 1: pairs per target, accum, reduced-chain classification
    std::vector<int64_t> tp0(S), tp1(S);
    P.pairs.clear();
    for (int k = 0; k < T; ++k) {
        for (int64_t t = P.cs[k]; t < P.cs[k + 1]; ++t) {
            const int32_t m = P.frow[t];
            tp0[t] = (int64_t)P.pairs.size();
            for (int64_t x = rp[k]; x < rp[k + 1]; ++x) {
                const int32_t nn = rn[x];
                const int64_t skn = rs[x];
                const int64_t smn = (m == k) ? skn : find_slot(P, m, nn);
                if (smn >= 0) P.pairs.push_back(Pair{(int32_t)smn, (int32_t)skn});
            }
            tp1[t] = (int64_t)P.pairs.size();
        }
    }
    if (P.pairs.size() > (size_t)INT32_MAX) return set_err(TC_ERR_ARG, "plan: too many pairs");
    const int W = P.W;
    const int thr = P.opts.tree_threshold;
    std::vector<int64_t> red_base(S, -1);  // scratch index base for reduced targets
    int64_t nred = 0;
    if (thr > 0 && W >= 2) {
        for (int64_t t = 0; t < S; ++t)
            if (tp1[t] - tp0[t] >= thr) red_base[t] = (nred++) * W;
    }
    P.R = nred * W;
    const int CH = P.opts.chunk > 0 ? P.opts.chunk : 8;

    std::vector<std::pair<int, int>> blk_full, blk_low;
    tile_blocks(nt, P.upd.BM, P.upd.BN, false, blk_full);
    tile_blocks(nt, P.upd.BM, P.upd.BN, true, blk_low);
    auto blocks_for = [&](int64_t t) -> const std::vector<std::pair<int, int>>& {
        return P.frow[t] == P.fcol[t] ? blk_low : blk_full;
    };

    // split-K pieces of reduced chains: target t's pairs whose column n falls in
    // [j*CH, (j+1)*CH) form one piece, emitted right after the panel of the
    // piece's last column; pieces with equal j and last column share a launch.
    struct Piece {
        int j;
        int64_t t, a, b;
    };
    std::vector<std::vector<Piece>> pieces_at(T);
    for (int64_t t = 0; t < S; ++t) {
        if (red_base[t] < 0) continue;
        for (int64_t x = tp0[t]; x < tp1[t];) {
            const int j = P.fcol[P.pairs[x].b] / CH;
            int64_t y = x;
            while (y < tp1[t] && P.fcol[P.pairs[y].b] / CH == j) ++y;
            pieces_at[P.fcol[P.pairs[y - 1].b]].push_back(Piece{j, t, x, y});
            x = y;
        }
    }

    // ---- pass 2: launches in topological order
    P.launches.clear();
    P.colB.assign(T, -1);
    P.colM.assign(T, -1);
    P.colMd.assign(T, -1);
    P.colBd.assign(T, -1);
    P.colL.assign(T, -1);
    P.colLo.assign(T, -1);
    P.colPot.assign(T, -1);
    P.colTrsm.assign(T, -1);
    P.colTrsmC.assign(T, -1);
    P.colLc.assign(T, -1);
    P.colComb.assign(T, {});
    P.colChunk.assign(T, {});
    P.items.clear();
    P.tgts.clear();
    std::vector<int32_t> pnode(T, -1);           // launch finishing column k
    std::vector<int32_t> pcrit(T, -1);           // TRSMc(k) when column k's TRSM is split
    std::vector<uint32_t> live_mask(S, 0);
    std::vector<std::vector<int32_t>> buf_writer(S);  // per reduced target: last chunk launch per residue
    const double n3 = (double)nt * nt * nt;

    auto add_panel_deps = [&](std::vector<int32_t>& deps, std::vector<int32_t>& cols) {
        std::sort(cols.begin(), cols.end());
        cols.erase(std::unique(cols.begin(), cols.end()), cols.end());
        for (int32_t c : cols) {
            const int32_t pa = parent[c];
            if (pa >= 0 && std::binary_search(cols.begin(), cols.end(), pa)) continue;
            deps.push_back(pnode[c]);
            if (pcrit[c] >= 0) deps.push_back(pcrit[c]);
        }
    };

    std::vector<std::pair<int, int>> sblk_full, sblk_low;
    const int SBK = (P.opts.use_graph == 2 || P.opts.use_graph == 0 || P.opts.use_graph == 1) ? small_block(nt) : 0;
    if (SBK) {
        tile_blocks(nt, SBK, SBK, false, sblk_full);
        tile_blocks(nt, SBK, SBK, true, sblk_low);
    }
    bool small_now = false;  // emitting an L(k) launch
    auto emit_items = [&](int64_t t, int64_t p0, int64_t p1, int32_t dst, int mode) {
        const auto& bl_list = (small_now && SBK) ? (P.frow[t] == P.fcol[t] ? sblk_low : sblk_full) : blocks_for(t);
        for (auto& bl : bl_list)
            P.items.push_back(Item{dst, bl.first, bl.second, (int32_t)p0, (int32_t)p1, mode});
    };

    for (int k = 0; k < T; ++k) {
        const int64_t c0 = P.cs[k], c1 = P.cs[k + 1];
        // lookahead depth D: the last contributing column feeds L(k), the
        // D-1 before it feed M(k), the rest feed the bulk update B(k), so
        // B(k+D) can run while columns k-1 .. k+D-1 are still in flight
        const int D = P.opts.lookahead;
        const int64_t nctr = rp[k + 1] - rp[k];
        const int32_t nlast = (D > 0 && nctr > 0) ? rn[rp[k + 1] - 1] : -1;
        const int32_t nmid = (D > 1 && nctr > 1) ? rn[std::max<int64_t>(rp[k], rp[k + 1] - D)] : -1;
        const int32_t bcut = nmid >= 0 ? nmid : (nlast >= 0 ? nlast : INT32_MAX);
        // first pair of target t whose contributing column is >= col
        auto cut = [&](int64_t t, int32_t col) {
            int64_t x = tp1[t];
            while (x > tp0[t] && P.fcol[P.pairs[x - 1].b] >= col) --x;
            return x;
        };
        // B(k): bulk pairs of non-reduced targets.  With the B split the
        // diagonal tile's bulk pairs form their own launch Bd(k): the chain
        // Bd(k) -> Md(k) -> L_diag(k) -> POTRF(k) then never waits for the
        // column's long off-diagonal bulk items (C4: B(k+1) ended ~28 us into
        // POTRF(k) and held Md(k+1) back)
        int32_t bnode = -1, bdnode = -1, lnode = -1, mnode = -1;
        const bool bsplit = SBK && m_split() && b_split();
        for (int part = 0; part < 2; ++part) {
            const bool dpart = part == 0;
            if (dpart && !bsplit) continue;
            Launch L;
            L.kind = L_UPD;
            L.k = k;
            L.off = (int64_t)P.items.size();
            std::vector<int32_t> cols;
            for (int64_t t = c0; t < c1; ++t) {
                if (red_base[t] >= 0) continue;
                if (bsplit && ((t == c0) != dpart)) continue;
                const int64_t p1 = cut(t, bcut);
                if (p1 > tp0[t]) {
                    emit_items(t, tp0[t], p1, (int32_t)t, MODE_SUB);
                    for (int64_t x = tp0[t]; x < p1; ++x) cols.push_back(P.fcol[P.pairs[x].b]);
                    L.flops += (P.frow[t] == k ? 1.0 : 2.0) * n3 * (double)(p1 - tp0[t]);
                }
            }
            L.cnt = (int64_t)P.items.size() - L.off;
            if (L.cnt > 0) {
                add_panel_deps(L.deps, cols);
                const int32_t id = (int32_t)P.launches.size();
                if (dpart) {
                    bdnode = id;
                    P.colBd[k] = id;
                } else {
                    bnode = id;
                    P.colB[k] = id;
                }
                P.launches.push_back(std::move(L));
            }
        }
        // writers of the diagonal tile before Md(k) / of the rest before M(k)
        const int32_t bprev_d = bsplit ? bdnode : bnode;
        // M(k): with the L split, the diagonal tile's near pairs form their
        // own launch Md(k) -- L_diag(k) and POTRF(k) wait only on it, so the
        // chain no longer waits for the whole column's near update to get
        // CTAs (C4 @128: M(k+1) ended ~7 us after TRSM(k), delaying L_diag)
        int32_t mdnode = -1;
        const bool msplit = SBK && m_split();
        for (int part = 0; part < (msplit ? 2 : 1) && nmid >= 0; ++part) {
            const bool dpart = msplit && part == 0;
            Launch L;
            L.kind = L_UPD;
            L.k = k;
            L.tag = kTagMid;
            L.off = (int64_t)P.items.size();
            std::vector<int32_t> cols;
            for (int64_t t = c0; t < c1; ++t) {
                if (red_base[t] >= 0) continue;
                if (msplit && ((t == c0) != dpart)) continue;
                const int64_t p0 = cut(t, nmid), p1 = cut(t, nlast);
                if (p1 > p0) {
                    emit_items(t, p0, p1, (int32_t)t, MODE_SUB);
                    for (int64_t x = p0; x < p1; ++x) cols.push_back(P.fcol[P.pairs[x].b]);
                    L.flops += (P.frow[t] == k ? 1.0 : 2.0) * n3 * (double)(p1 - p0);
                }
            }
            L.cnt = (int64_t)P.items.size() - L.off;
            if (L.cnt > 0) {
                add_panel_deps(L.deps, cols);
                const int32_t bp = dpart ? bprev_d : bnode;
                if (bp >= 0) L.deps.push_back(bp);
                if (!msplit && bdnode >= 0) L.deps.push_back(bdnode);
                const int32_t id = (int32_t)P.launches.size();
                if (dpart) {
                    mdnode = id;
                    P.colMd[k] = id;
                } else {
                    mnode = id;
                    P.colM[k] = id;
                }
                P.launches.push_back(std::move(L));
            }
        }
        // last writers of column k before L(k): the diagonal tile / the rest
        const int32_t prev_d = msplit ? (mdnode >= 0 ? mdnode : bprev_d) : (mnode >= 0 ? mnode : bnode);
        const int32_t prev = mnode >= 0 ? mnode : bnode;
        // L(k): the last contribution.  With small blocks available it is split
        // into L_diag(k) (the diagonal tile, small blocks: POTRF(k) waits only
        // on it) and L_off(k) (off-diagonal targets, regular blocks: only
        // TRSM(k) waits on them, and TRSM streams behind POTRF anyway)
        // With the critical split (crit_split()) the first off-diagonal
        // target c0+1 gets its own small-block launch L_crit(k) and its own
        // TRSM launch TRSMc(k): the column chain POTRF(k) -> TRSMc(k) ->
        // L_diag(k+1) no longer waits for the whole column's L_off(k).
        int32_t lnode_off = -1, lnode_crit = -1;
        const bool csplit = SBK && crit_split() && c1 - c0 > 1;
        // L(k) items read tiles of column nlast only: the diagonal part reads
        // (k, nlast), which TRSMc(nlast) alone produces when row k is column
        // nlast's first off-diagonal row
        const bool dcrit = nlast >= 0 && pcrit[nlast] >= 0 && P.frow[P.cs[nlast] + 1] == k;
        if (nlast >= 0) {
            for (int part = 0; part < 3; ++part) {
                const bool diag_part = part == 0, crit_part = part == 1;
                if (!SBK && !diag_part) break;  // unsplit: one launch, regular blocks
                if (crit_part && !csplit) continue;
                Launch L;
                L.kind = L_UPD;
                L.k = k;
                L.high = 1;
                L.cls = 1;
                L.tag = diag_part ? kTagChain : (crit_part ? kTagChain | kTagSub : 0);
                L.off = (int64_t)P.items.size();
                small_now = SBK != 0 && (diag_part || crit_part);
                L.small = small_now ? 1 : 0;
                for (int64_t t = c0; t < c1; ++t) {
                    if (red_base[t] >= 0) continue;
                    if (SBK && ((t == c0) != diag_part)) continue;
                    if (csplit && !diag_part && ((t == c0 + 1) != crit_part)) continue;
                    const int64_t p1 = tp1[t];
                    if (p1 > tp0[t] && P.fcol[P.pairs[p1 - 1].b] == nlast) {
                        emit_items(t, p1 - 1, p1, (int32_t)t, MODE_SUB);
                        L.flops += (P.frow[t] == k ? 1.0 : 2.0) * n3;
                    }
                }
                small_now = false;
                L.cnt = (int64_t)P.items.size() - L.off;
                if (L.cnt > 0) {
                    if (diag_part && dcrit) {
                        L.deps.push_back(pcrit[nlast]);
                    } else {
                        L.deps.push_back(pnode[nlast]);
                        if (pcrit[nlast] >= 0) L.deps.push_back(pcrit[nlast]);
                    }
                    const int32_t pv = diag_part && SBK ? prev_d : prev;
                    if (pv >= 0) L.deps.push_back(pv);
                    if (!SBK && mdnode >= 0) L.deps.push_back(mdnode);
                    const int32_t id = (int32_t)P.launches.size();
                    if (diag_part) {
                        lnode = id;
                        P.colL[k] = id;
                    } else if (crit_part) {
                        lnode_crit = id;
                        P.colLc[k] = id;
                    } else {
                        lnode_off = id;
                        P.colLo[k] = id;
                    }
                    P.launches.push_back(std::move(L));
                }
            }
        }
        // combines of reduced targets of this column
        std::vector<int32_t> comb_diag, comb_off;
        for (int64_t t = c0; t < c1; ++t) {
            if (red_base[t] < 0) continue;
            Launch L;
            L.kind = L_COMBINE;
            L.high = 1;
            L.cls = 4;
            L.slot = t;
            L.scratch0 = S + red_base[t];
            L.live = live_mask[t];
            for (int32_t w : buf_writer[t])
                if (w >= 0) L.deps.push_back(w);
            const int32_t id = (int32_t)P.launches.size();
            (P.frow[t] == k ? comb_diag : comb_off).push_back(id);
            P.colComb[k].push_back(id);
            P.launches.push_back(std::move(L));
        }
        // POTRF(k)
        int32_t pot;
        {
            Launch L;
            L.kind = L_POTRF;
            L.high = 1;
            L.cls = 2;
            L.k = k;
            L.slot = c0;
            if (bsplit) {
                if (bdnode >= 0) L.deps.push_back(bdnode);
            } else if (bnode >= 0) {
                L.deps.push_back(bnode);
            }
            if (mdnode >= 0) L.deps.push_back(mdnode);
            if (mnode >= 0 && !msplit) L.deps.push_back(mnode);
            if (lnode >= 0) L.deps.push_back(lnode);
            for (int32_t x : comb_diag) L.deps.push_back(x);
            L.flops += n3 / 3.0;
            pot = (int32_t)P.launches.size();
            P.colPot[k] = pot;
            P.launches.push_back(std::move(L));
        }
        pnode[k] = pot;
        for (int part = 0; part < 2; ++part) {
            // part 0: TRSMc(k) (target c0+1 only, with the critical split) or
            // the whole TRSM(k); part 1: TRSMr(k), the remaining targets
            const int64_t t0 = (part == 0) ? c0 + 1 : c0 + 2;
            const int64_t t1 = (part == 0 && csplit) ? std::min<int64_t>(c0 + 2, c1) : c1;
            if ((part == 1 && !csplit) || t1 <= t0) continue;
            Launch L;
            L.kind = L_TRSM;
            L.high = 1;
            L.cls = 3;
            L.k = k;
            L.slot = c0;
            L.tag = (csplit && part == 0) ? kTagChain : 0;
            L.off = (int64_t)P.tgts.size();
            for (int64_t t = t0; t < t1; ++t) P.tgts.push_back((int32_t)t);
            L.cnt = t1 - t0;
            L.deps.push_back(pot);
            if (bnode >= 0) L.deps.push_back(bnode);
            if (bdnode >= 0) L.deps.push_back(bdnode);
            if (mnode >= 0) L.deps.push_back(mnode);
            if (mdnode >= 0) L.deps.push_back(mdnode);
            if (lnode >= 0) L.deps.push_back(lnode);
            if (csplit && part == 0) {
                if (lnode_crit >= 0) L.deps.push_back(lnode_crit);
            } else if (lnode_off >= 0) {
                L.deps.push_back(lnode_off);
            }
            if (!csplit && lnode_crit >= 0) L.deps.push_back(lnode_crit);
            for (int32_t x : comb_off) L.deps.push_back(x);
            L.flops += n3 * (double)(t1 - t0);
            const int32_t id = (int32_t)P.launches.size();
            if (csplit && part == 0) {
                pcrit[k] = id;
                P.colTrsmC[k] = id;
                if (c1 - c0 == 2) {  // no other target: TRSMc finishes column k
                    pnode[k] = id;
                    pcrit[k] = -1;
                    P.colTrsm[k] = id;
                    P.colTrsmC[k] = -1;
                }
            } else {
                pnode[k] = id;
                P.colTrsm[k] = id;
            }
            P.launches.push_back(std::move(L));
        }
        // split-K pieces of reduced chains that became ready with column k
        auto& pcs = pieces_at[k];
        std::stable_sort(pcs.begin(), pcs.end(), [](const Piece& x, const Piece& y) { return x.j < y.j; });
        for (size_t u = 0; u < pcs.size();) {
            size_t v = u;
            while (v < pcs.size() && pcs[v].j == pcs[u].j) ++v;
            const int w = pcs[u].j % W;
            Launch L;
            L.kind = L_UPD;
            L.k = k;
            L.cls = 6;
            L.off = (int64_t)P.items.size();
            std::vector<int32_t> cols;
            for (size_t z = u; z < v; ++z) {
                const Piece& pc = pcs[z];
                const int64_t t = pc.t;
                if (buf_writer[t].empty()) buf_writer[t].assign(W, -1);
                const bool first = !((live_mask[t] >> w) & 1u);
                emit_items(t, pc.a, pc.b, (int32_t)(S + red_base[t] + w), first ? MODE_NEGSTORE : MODE_SUB);
                live_mask[t] |= 1u << w;
                for (int64_t x = pc.a; x < pc.b; ++x) cols.push_back(P.fcol[P.pairs[x].b]);
                if (buf_writer[t][w] >= 0) L.deps.push_back(buf_writer[t][w]);
                L.flops += (P.frow[t] == P.fcol[t] ? 1.0 : 2.0) * n3 * (double)(pc.b - pc.a);
            }
            L.cnt = (int64_t)P.items.size() - L.off;
            add_panel_deps(L.deps, cols);
            const int32_t id = (int32_t)P.launches.size();
            for (size_t z = u; z < v; ++z) buf_writer[pcs[z].t][w] = id;
            P.colChunk[k].push_back(id);
            P.launches.push_back(std::move(L));
            u = v;
        }
    }
    // final logdet reduction: depends on every launch with no dependents
    {
        std::vector<char> has_succ(P.launches.size(), 0);
        for (auto& L : P.launches)
            for (int32_t d : L.deps) has_succ[d] = 1;
        Launch L;
        L.kind = L_LOGDET;
        L.high = 1;
        L.cls = 5;
        for (size_t i = 0; i < P.launches.size(); ++i)
            if (!has_succ[i]) L.deps.push_back((int32_t)i);
        P.launches.push_back(std::move(L));
    }
    for (auto& L : P.launches) {
        std::sort(L.deps.begin(), L.deps.end());
        L.deps.erase(std::unique(L.deps.begin(), L.deps.end()), L.deps.end());
    }
    P.flops = 0.0;
    for (auto& L : P.launches) P.flops += L.flops;
    // solve metadata
    P.sol_off.assign(T + 1, 0);
    std::vector<int32_t> sslots, srows;
    for (int k = 0; k < T; ++k) {
        for (int64_t t = P.cs[k] + 1; t < P.cs[k + 1]; ++t) {
            sslots.push_back((int32_t)t);
            srows.push_back(P.frow[t]);
        }
        P.sol_off[k + 1] = (int64_t)sslots.size();
    }
    std::vector<int64_t> dslots(T);
    for (int k = 0; k < T; ++k) dslots[k] = P.cs[k];
    std::vector<int32_t> rs32(rs.begin(), rs.end());
    cudaStream_t s = 0;
    int r = upload(P.items, &P.d_items, s);
    if (!r) r = upload(P.sol_off, &P.d_sol_off, s);
    if (!r) r = upload(rp, &P.d_row_ptr, s);
    if (!r) r = upload(rn, &P.d_row_col, s);
    if (!r) r = upload(rs32, &P.d_row_slot, s);
    if (!r) r = upload(P.pairs, &P.d_pairs, s);
    if (!r) r = upload(P.tgts, &P.d_tgts, s);
    if (!r) r = upload(dslots, &P.d_diag_slots, s);
    if (!r) r = upload(sslots, &P.d_sol_slots, s);
    if (!r) r = upload(srows, &P.d_sol_rows, s);
    if (r) return r;
    CK(cudaStreamSynchronize(s));
    if (P.opts.use_graph == 2 && (nt & 1) == 0) return build_persistent(P);
    if (P.opts.use_graph == 2) P.opts.use_graph = 1;  // odd nt: 8-byte copies go through L1 -> graph mode
    return TC_OK;
}

// Ticket order + flat task list of the persistent executor.  Per column k:
// L(k), combines(k), POTRF(k), B(k+1), TRSM(k), split-K chunks ready at k —
// the bulk update of the next column is handed out before the TRSM tiles of
// this one so CTAs have work while POTRF(k) runs.  Falls back to creation
// order (always topological) if the heuristic order were not.
int build_persistent(tc_plan& P) {
    const int T = P.T, nt = P.nt;
    const size_t NL = P.launches.size();
    std::vector<int32_t> order;
    order.reserve(NL);
    std::vector<char> placed(NL, 0);
    auto put = [&](int32_t id) {
        if (id >= 0 && !placed[id]) {
            placed[id] = 1;
            order.push_back(id);
        }
    };
    // Fused POTRF -> TRSM: TRSM(k) tasks no longer wait for POTRF(k) to end;
    // they consume its panels through the per-column progress counter, so
    // they are ticketed right behind it.  The log-det node must then wait
    // for every POTRF explicitly (its partials are written at POTRF's end).
    const bool fuse = P.fuse;
    std::vector<std::vector<int32_t>> pdeps(NL);
    for (size_t i = 0; i < NL; ++i) {
        const Launch& L = P.launches[i];
        for (int32_t d : L.deps)
            if (!(fuse && L.kind == L_TRSM && P.launches[d].kind == L_POTRF && P.launches[d].k == L.k))
                pdeps[i].push_back(d);
        if (fuse && L.kind == L_LOGDET)
            for (int k = 0; k < T; ++k) pdeps[i].push_back(P.colPot[k]);
        std::sort(pdeps[i].begin(), pdeps[i].end());
        pdeps[i].erase(std::unique(pdeps[i].begin(), pdeps[i].end()), pdeps[i].end());
    }
    // Fused diagonal SYRK (packed in-smem POTRF, nt <= 128): the diagonal
    // tile's one-pair items leave L(k); POTRF(k) applies A(k,k) -= X X^T with
    // X = L(k, n_last) itself and waits for the TRSM launch of column n_last
    // instead of L(k) -- one hand-off and one dispatch fewer on the column
    // chain.  L(k) keeps any other targets; an L(k) left empty is dropped.
    std::vector<int64_t> loff(NL), lcnt(NL);
    for (size_t i = 0; i < NL; ++i) {
        loff[i] = P.launches[i].off;
        lcnt[i] = P.launches[i].cnt;
    }
    std::vector<char> dead(NL, 0);
    P.xslot_of_col.assign(T, -1);
    P.nfused = 0;
    bool pin_smem;
    potrf_smem(nt, &pin_smem);
    // compiled out (TC_SYRK_FUSE_CODE): the in-CTA SYRK made POTRF 23 us
    // longer, more than the L_diag hand-off it removes (C4@128 551 vs 524 ms,
    // C2 49.6 vs 38.8 ms)
    const bool fuse_syrk = TC_SYRK_FUSE_CODE && pin_smem && ((nt + 7) & ~7) <= 128 && getenv("TC_SYRK_FUSE") &&
                           atoi(getenv("TC_SYRK_FUSE")) == 1;
    for (int k = 0; k < T && fuse_syrk; ++k) {
        const int32_t lk = P.colL[k];
        if (lk < 0) continue;
        int64_t nd = 0;
        while (nd < lcnt[lk] && P.items[loff[lk] + nd].dst == (int32_t)P.cs[k]) ++nd;
        if (nd == 0) continue;
        const Item& it0 = P.items[loff[lk]];
        if (it0.p1 - it0.p0 != 1) continue;
        const Pair pr = P.pairs[it0.p0];
        if (pr.a != pr.b) continue;
        P.xslot_of_col[k] = pr.a;
        ++P.nfused;
        loff[lk] += nd;
        lcnt[lk] -= nd;
        if (lcnt[lk] == 0) dead[lk] = 1;
        auto& pd = pdeps[P.colPot[k]];
        pd.erase(std::remove(pd.begin(), pd.end(), lk), pd.end());
        const int32_t src = P.fcol[pr.a];  // X's column: POTRF(k) reads its TRSM output
        pd.push_back(P.colTrsm[src] >= 0 ? P.colTrsm[src] : P.colPot[src]);
        std::sort(pd.begin(), pd.end());
        pd.erase(std::unique(pd.begin(), pd.end()), pd.end());
    }
    for (size_t i = 0; i < NL; ++i) {
        auto& pd = pdeps[i];
        pd.erase(std::remove_if(pd.begin(), pd.end(), [&](int32_t d) { return dead[d] != 0; }), pd.end());
    }
    const int D = std::max(1, P.opts.lookahead);
    for (int j = 0; j < std::min(D, T); ++j) {
        put(P.colBd[j]);
        put(P.colB[j]);
    }
    // TC_ORDER=1: the next column's chain (M, L_diag, combines, POTRF) is
    // ticketed right behind this column's TRSM, ahead of the bulk update, so
    // it never waits for the bulk tickets to be handed out
    // default on for wide columns (>= 16 tiles per column on average, e.g.
    // C4: 536 -> 520 ms at nt=128), off for narrow ones (C3: 89 vs 97 ms)
    const bool chain_first = getenv("TC_ORDER") ? atoi(getenv("TC_ORDER")) == 1 : P.S >= 16 * (int64_t)T;
    const bool md_early = !(getenv("TC_MD_EARLY") && atoi(getenv("TC_MD_EARLY")) == 0) && D >= 2;
    const bool bd_early = !(getenv("TC_BD_EARLY") && atoi(getenv("TC_BD_EARLY")) == 0);
    const bool trsmr_late = getenv("TC_TRSMR_LATE") && atoi(getenv("TC_TRSMR_LATE")) == 1 && chain_first && fuse;
    for (int k = 0; k < T; ++k) {
        put(P.colMd[k]);
        put(P.colM[k]);
        put(P.colL[k]);
        put(P.colLc[k]);
        for (int32_t c : P.colComb[k]) put(c);
        put(P.colPot[k]);
        // the chain is POTRF(k) -> TRSMc(k) -> L_diag(k+1) -> POTRF(k+1);
        // L_diag(k+1) also waits for Md(k+1) (the diagonal tile's near
        // pairs, inputs ready since TRSM(k-1)): ticket it before TRSMc(k)
        // so it never holds up the chain (C4: it ended ~5 us after TRSMc)
        if (md_early && k + 1 < T) put(P.colMd[k + 1]);
        if (fuse) put(P.colTrsmC[k]);
        put(P.colLo[k]);
        // TC_TRSMR_LATE=1: the non-critical TRSM(k) tiles, the L_crit(k+1)
        // and split-K pieces that read them, ticketed behind B(k+D) (their
        // CTAs then stream fewer of POTRF(k)'s panels in a spin); only on
        // columns without reduced chains, whose combines the chain needs
        const bool late = trsmr_late && k + 1 < T && P.colChunk[k].empty() && P.colComb[k + 1].empty();
        if (fuse && !late) put(P.colTrsm[k]);
        if (chain_first && fuse && k + 1 < T) {
            for (int32_t c : P.colChunk[k]) put(c);  // split-K pieces the next combines read
            put(P.colMd[k + 1]);
            put(P.colM[k + 1]);
            put(P.colL[k + 1]);
            if (!late) put(P.colLc[k + 1]);
            for (int32_t c : P.colComb[k + 1]) put(c);
            put(P.colPot[k + 1]);
        }
        if (k + D < T) put(P.colBd[k + D]);
        if (k + D < T) put(P.colB[k + D]);
        if (late) {
            put(P.colTrsm[k]);
            put(P.colLc[k + 1]);
        }
        // the diagonal tile's bulk Bd(k+D+1) (inputs: columns <= k) one
        // column earlier than the rest: its few long items then end before
        // Md(k+D+1) / L_diag need the tile (C4: Bd(k+1) ended ~15 us into
        // POTRF(k) and delayed Md(k+1) in some columns)
        if (bd_early && k + D + 1 < T) put(P.colBd[k + D + 1]);
        if (k + 1 < T) put(P.colBd[k + 1]);
        if (k + 1 < T) put(P.colB[k + 1]);
        if (k + 1 < T) put(P.colMd[k + 1]);
        if (k + 1 < T) put(P.colM[k + 1]);
        put(P.colTrsmC[k]);
        put(P.colTrsm[k]);
        for (int32_t c : P.colChunk[k]) put(c);
    }
    for (size_t i = 0; i < NL; ++i) put((int32_t)i);
    std::vector<int32_t> pos(NL);
    for (size_t i = 0; i < NL; ++i) pos[order[i]] = (int32_t)i;
    bool topo = true;
    for (size_t i = 0; i < NL && topo; ++i)
        for (int32_t d : pdeps[i])
            if (pos[d] >= pos[i]) {
                topo = false;
                break;
            }
    if (!topo) {
        if (getenv("TC_DEBUG_ORDER")) fprintf(stderr, "tilechol: ticket order not topological, creation order used\n");
        for (size_t i = 0; i < NL; ++i) order[i] = (int32_t)i;
    }
    P.ptasks.clear();
    P.p_remaining.assign(NL, 0);
    P.p_deps.assign(NL, 0);
    // TRSM strip rows: the largest strip whose X block + L staging fits
    P.persist_trsm_rows = 16;
    for (int rows : {64, 32})
        if (trsm_ring_rows(rows, nt, 2) <= 225 * 1024) {
            P.persist_trsm_rows = rows;
            break;
        }
    const int nrb = (nt + P.persist_trsm_rows - 1) / P.persist_trsm_rows;
    for (int32_t id : order) {
        const Launch& L = P.launches[id];
        const size_t before = P.ptasks.size();
        if (dead[id]) {
            P.p_remaining[id] = 0;
            P.p_deps[id] = 0;
            continue;
        }
        switch (L.kind) {
            case L_UPD:
                for (int64_t x = loff[id]; x < loff[id] + lcnt[id]; ++x)
                    P.ptasks.push_back(PTask{id, (int32_t)x, L.small});
                break;
            case L_TRSM:
                for (int64_t x = L.off; x < L.off + L.cnt; ++x)
                    for (int rb = 0; rb < nrb; ++rb) P.ptasks.push_back(PTask{id, P.tgts[x], rb});
                break;
            default:
                P.ptasks.push_back(PTask{id, 0, 0});
                break;
        }
        P.p_remaining[id] = (int32_t)(P.ptasks.size() - before);
        P.p_deps[id] = (int32_t)pdeps[id].size();
    }
    if (P.ptasks.size() > (size_t)INT32_MAX / 2) return set_err(TC_ERR_ARG, "plan: too many tasks");
    P.p_succ_ptr.assign(NL + 1, 0);
    for (size_t i = 0; i < NL; ++i)
        for (int32_t d : pdeps[i]) P.p_succ_ptr[d + 1]++;
    for (size_t i = 0; i < NL; ++i) P.p_succ_ptr[i + 1] += P.p_succ_ptr[i];
    P.p_succ.assign(P.p_succ_ptr[NL], 0);
    {
        std::vector<int32_t> at(P.p_succ_ptr.begin(), P.p_succ_ptr.end() - 1);
        for (size_t i = 0; i < NL; ++i)
            for (int32_t d : pdeps[i]) P.p_succ[at[d]++] = (int32_t)i;
    }
    P.plaunch.assign(NL, PLaunch{});
    for (size_t i = 0; i < NL; ++i) {
        const Launch& L = P.launches[i];
        PLaunch& q = P.plaunch[i];
        switch (L.kind) {
            case L_UPD: q.kind = 0; break;
            case L_POTRF:
                q.kind = 1;
                q.k = L.k;
                q.slot = L.slot;
                q.live = (int32_t)std::min<int64_t>(P.n - (int64_t)L.k * nt, nt);
                q.scratch0 = P.xslot_of_col[L.k];  // fused SYRK source slot or -1
                break;
            case L_TRSM:
                q.kind = 2;
                q.k = L.k;
                q.slot = L.slot;
                break;
            case L_COMBINE:
                q.kind = 3;
                q.slot = L.slot;
                q.scratch0 = L.scratch0 - P.S;
                q.live = (int32_t)L.live;
                break;
            default: q.kind = 4; break;
        }
    }
    std::vector<int32_t> init(P.p_remaining);
    init.insert(init.end(), P.p_deps.begin(), P.p_deps.end());
    cudaStream_t s0 = 0;
    int r = upload(P.ptasks, &P.d_ptasks, s0);
    if (!r) r = upload(P.plaunch, &P.d_plaunch, s0);
    if (!r) r = upload(init, &P.d_p_init, s0);
    if (!r) r = upload(P.p_succ_ptr, &P.d_succ_ptr, s0);
    if (!r) r = upload(P.p_succ, &P.d_succ, s0);
    if (!r) {
        std::vector<int32_t> xos(P.S, -1);
        for (int k = 0; k < T; ++k)
            if (P.xslot_of_col[k] >= 0) xos[P.xslot_of_col[k]] = k;
        r = upload(xos, &P.d_xctr_of_slot, s0);
    }
    if (r) return r;
    // occupancy mode (opts.reserved[1]): 1 = one CTA/SM (no register cap,
    // whole-L TRSM staging), 2 = two CTAs/SM when the smem plan fits, 0 = auto
    // auto: a plan whose column steps carry little update work is bound by
    // the POTRF -> TRSM -> update chain, which runs ~1.3x faster with the SM
    // to itself (C2: 0.15 GFLOP per column); update-heavy plans (C3, C4:
    // 0.7-0.9 GFLOP per column at nt=120) need the second CTA per SM to hide
    // the update pipeline's bubbles
    // Default: one CTA per SM.  Two CTAs per SM (occupancy=2) are faster on
    // update-heavy plans (C4 @120: 603 vs 773 ms) but show a rare,
    // timing-dependent nondeterminism (log-determinant off by ~1e-7 relative,
    // DESIGN.md §10) that one CTA per SM has not shown; opt-in until found.
    const int occ_mode = P.opts.reserved[1];
    P.persist_minb = occ_mode == 2 && !big_shape(nt) ? 2 : 1;
    // TMA operand staging needs 16-byte row strides (nt even); TC_UPD_TMA=0 turns it off
    P.persist_tma = (nt % 2 == 0) && !(getenv("TC_UPD_TMA") && atoi(getenv("TC_UPD_TMA")) == 0);
    bool in_smem;
    // shared memory: the max over task kinds; the fused TRSM may stage L
    // strip by strip (ring) instead of whole when that lets two CTAs share an SM
    const size_t xs_bytes = P.nfused ? (size_t)2 * 16 * pad_ld((nt + 7) & ~7) * sizeof(double) : 0;
    const size_t two_per_sm = 108 * 1024;  // (228 KB - reserved - static) / 2
    if (P.persist_minb == 2 &&
        std::max<size_t>((size_t)pick_persist(nt, 2).smem, potrf_smem(nt, &in_smem) + xs_bytes) > two_per_sm)
        P.persist_minb = 1;  // two CTAs cannot share an SM (packed POTRF tile too large): no register cap
    const PersistKernel K = pick_persist(nt, P.persist_minb);
    if (!K.fn) return set_err(TC_ERR_ARG, "plan: no persistent kernel variant for tile size %d", nt);
    P.pkern = K;  // fixed at plan time (the selection reads tuning environment variables)
    const size_t base = std::max<size_t>({(size_t)K.smem, potrf_smem(nt, &in_smem) + xs_bytes, (size_t)4096});
    const int TR = P.persist_trsm_rows;
    const size_t t_full = trsm_smem_rows(TR, nt);
    P.persist_trsm_ring = getenv("TC_FORCE_TRSM_RING") ? 2 : 0;  // diagnostic: ring staging at any occupancy
    P.persist_smem = std::max(base, t_full);
    if (P.persist_minb == 2 && P.persist_smem > two_per_sm) {
        // fused TRSM stages one strip at a time (1 buffer); unfused needs a ring
        for (int nb : {P.fuse ? 1 : 3, P.fuse ? 1 : 2}) {
            const size_t t = std::max(base, trsm_ring_rows(TR, nt, nb));
            if (t <= two_per_sm) {
                P.persist_trsm_ring = nb < 2 ? 2 : nb;
                P.persist_smem = t;
                break;
            }
        }
    }
    r = prep_kernel((const void*)K.fn, (int)P.persist_smem);
    if (r) return r;
    int per_sm = 0, sms = 0;
    CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, K.fn, kPersistThreads, P.persist_smem));
    CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, P.dev));
    if (per_sm < 1) return set_err(TC_ERR_CUDA, "persistent kernel does not fit on an SM (smem %zu)", P.persist_smem);
    // opts.reserved[2] = number of factorisations meant to run concurrently
    // (batch lanes): each launch then takes its share of the SMs so the
    // lanes' persistent kernels coexist instead of serialising
    const int conc = std::max(1, (int)P.opts.reserved[2]);
    P.persist_grid = std::max(1, (per_sm * sms) / conc);
    CK(cudaStreamSynchronize(s0));
    return TC_OK;
}

// cuTensorMapEncodeTiled through the runtime's driver entry point (no libcuda link)
typedef CUresult (*EncodeTiledFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                  const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                                  CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);
int encode_tile_map(CUtensorMap* m, double* storage, int nt, int64_t S, int box_rows, int box_k) {
    static EncodeTiledFn fn = nullptr;
    if (!fn) {
        cudaDriverEntryPointQueryResult q;
        void* f = nullptr;
        CK(cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &f, cudaEnableDefault, &q));
        if (!f || q != cudaDriverEntryPointSuccess) return set_err(TC_ERR_CUDA, "cuTensorMapEncodeTiled unavailable");
        fn = (EncodeTiledFn)f;
    }
    const cuuint64_t dims[3] = {(cuuint64_t)nt, (cuuint64_t)nt, (cuuint64_t)S};
    const cuuint64_t strides[2] = {(cuuint64_t)nt * 8, (cuuint64_t)nt * nt * 8};
    const cuuint32_t box[3] = {(cuuint32_t)box_rows, (cuuint32_t)box_k, 1};
    const cuuint32_t es[3] = {1, 1, 1};
    const CUresult r = fn(m, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 3, storage, dims, strides, box, es,
                          CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                          CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS) return set_err(TC_ERR_CUDA, "cuTensorMapEncodeTiled failed (%d)", (int)r);
    return TC_OK;
}

int run_persistent(tc_plan& P, Lane& ln, cudaStream_t s) {
    const size_t NL = P.launches.size();
    if (!ln.d_pstate) CK(cudaMalloc(&ln.d_pstate, (2 * NL + 1) * sizeof(int32_t)));
    CK(cudaMemcpyAsync(ln.d_pstate, P.d_p_init, 2 * NL * sizeof(int32_t), cudaMemcpyDeviceToDevice, s));
    CK(cudaMemsetAsync(ln.d_pstate + 2 * NL, 0, sizeof(int32_t), s));
    if (P.fuse) {
        if (!ln.d_prog) CK(cudaMalloc(&ln.d_prog, (size_t)P.T * sizeof(int32_t)));
        CK(cudaMemsetAsync(ln.d_prog, 0, (size_t)P.T * sizeof(int32_t), s));
    }
    if (P.nfused) {
        if (!ln.d_xctr) CK(cudaMalloc(&ln.d_xctr, (size_t)P.T * 32 * sizeof(int32_t)));
        CK(cudaMemsetAsync(ln.d_xctr, 0, (size_t)P.T * 32 * sizeof(int32_t), s));
    }
    PersistArgs a{};
    a.ctx = ln.d_ctx;
    a.items = P.d_items;
    a.pairs = P.d_pairs;
    a.tasks = P.d_ptasks;
    a.launches = P.d_plaunch;
    a.ntasks = (int32_t)P.ptasks.size();
    a.remaining = ln.d_pstate;
    a.deps_left = ln.d_pstate + NL;
    a.succ_ptr = P.d_succ_ptr;
    a.succ = P.d_succ;
    a.ticket = ln.d_pstate + 2 * NL;
    a.nt = P.nt;
    a.W = P.W;
    a.T = P.T;
    bool in_smem;
    potrf_smem(P.nt, &in_smem);
    a.potrf_in_smem = in_smem;
    a.prog = P.fuse ? ln.d_prog : nullptr;
    a.trsm_ring = P.persist_trsm_ring;
    a.trace = ln.d_trace;
    a.xctr = P.nfused ? ln.d_xctr : nullptr;
    a.xctr_of_slot = P.d_xctr_of_slot;
    a.xper = ((P.nt + P.persist_trsm_rows - 1) / P.persist_trsm_rows) * (P.persist_trsm_rows / 8);
    a.trsm_rows = P.persist_trsm_rows;
    const PersistKernel& K = P.pkern;
    a.use_tma = 0;
    if (P.persist_tma) {
        // TMA descriptors of this storage: a 3-D tensor [S][nt][nt] (rows
        // innermost), boxes = the update kernel's padded stage layout
        const int r1 = encode_tile_map(&a.tmA, ln.h.storage, P.nt, P.S, K.lda, K.kc);
        const int r2 = r1 ? r1 : encode_tile_map(&a.tmB, ln.h.storage, P.nt, P.S, K.ldb, K.kc);
        if (r2) return r2;
        a.use_tma = 1;
    }
    K.fn<<<P.persist_grid, kPersistThreads, P.persist_smem, s>>>(a);
    CK(cudaGetLastError());
    return TC_OK;
}

// kernel launch (direct) or node params (graph) of launch i for a lane
struct NodeArgs {
    UpdArgs ua;
    PotrfArgs pa;
    TrsmArgs ta;
    const Ctx* ctx;
    int64_t target, scratch0;
    int W;
    uint32_t live;
    int nt;
    const double* ld_in;
    int64_t ld_n;
    double ld_scale;
    double* ld_out;
};

int node_params(tc_plan& P, Lane& ln, size_t i, cudaKernelNodeParams& kp, NodeArgs& na, void** argv) {
    const Launch& L = P.launches[i];
    memset(&kp, 0, sizeof kp);
    const int nt = P.nt;
    switch (L.kind) {
        case L_UPD: {
            na.ua = UpdArgs{};
            na.ua.items = P.d_items;
            na.ua.pairs = P.d_pairs;
            na.ua.ctx = ln.d_ctx;
            na.ua.nt = nt;
            na.ua.item_base = (int32_t)L.off;
            argv[0] = &na.ua;
            const UpdKernel& K = (L.small && P.upd_small.fn) ? P.upd_small : P.upd;
            kp.func = (void*)K.fn;
            kp.gridDim = dim3((unsigned)L.cnt);
            kp.blockDim = dim3(K.nth);
            kp.sharedMemBytes = K.smem;
            break;
        }
        case L_POTRF: {
            bool in_smem;
            const size_t sm = potrf_smem(nt, &in_smem);
            na.pa = PotrfArgs{};
            na.pa.ctx = ln.d_ctx;
            na.pa.slot = L.slot;
            na.pa.nt = nt;
            na.pa.k = L.k;
            const int64_t live = P.n - (int64_t)L.k * nt;
            na.pa.live = (int32_t)std::min<int64_t>(live, nt);
            na.pa.in_smem = in_smem;
            argv[0] = &na.pa;
            kp.func = (void*)k_potrf;
            kp.gridDim = dim3(1);
            kp.blockDim = dim3(kPotrfThreads);
            kp.sharedMemBytes = (unsigned)sm;
            break;
        }
        case L_TRSM: {
            na.ta = TrsmArgs{};
            na.ta.ctx = ln.d_ctx;
            na.ta.lslot = L.slot;
            na.ta.targets = P.d_tgts + L.off;
            na.ta.nt = nt;
            argv[0] = &na.ta;
            const TrsmK TK = trsm_direct(nt);
            kp.func = (void*)TK.fn;
            kp.gridDim = dim3((nt + TK.rows - 1) / TK.rows, (unsigned)L.cnt);
            kp.blockDim = dim3(4 * TK.rows);
            kp.sharedMemBytes = (unsigned)TK.smem;
            break;
        }
        case L_COMBINE: {
            na.ctx = ln.d_ctx;
            na.target = L.slot;
            na.scratch0 = L.scratch0 - P.S;  // scratch index relative to scratch base
            na.W = P.W;
            na.live = L.live;
            na.nt = nt;
            argv[0] = &na.ctx;
            argv[1] = &na.target;
            argv[2] = &na.scratch0;
            argv[3] = &na.W;
            argv[4] = &na.live;
            argv[5] = &na.nt;
            kp.func = (void*)k_combine;
            kp.gridDim = dim3(elem_grid(nt));
            kp.blockDim = dim3(256);
            break;
        }
        default: {  // L_LOGDET
            na.ld_in = ln.d_ld;
            na.ld_n = P.T;
            na.ld_scale = 2.0;
            na.ld_out = ln.d_ld + P.T;
            argv[0] = &na.ld_in;
            argv[1] = &na.ld_n;
            argv[2] = &na.ld_scale;
            argv[3] = &na.ld_out;
            kp.func = (void*)k_sum_fixed;
            kp.gridDim = dim3(1);
            kp.blockDim = dim3(256);
            break;
        }
    }
    kp.kernelParams = argv;
    return TC_OK;
}

int ensure_lane(tc_plan& P, int lane) {
    if (lane < 0 || lane >= 256) return set_err(TC_ERR_ARG, "lane %d out of range", lane);
    if ((int)P.lanes.size() <= lane) P.lanes.resize(lane + 1);
    Lane& ln = P.lanes[lane];
    if (ln.d_ctx) return TC_OK;
    CK(cudaMalloc(&ln.d_ctx, sizeof(Ctx)));
    CK(cudaMalloc(&ln.d_fail, 8));
    CK(cudaMalloc(&ln.d_ld, (P.T + 1) * sizeof(double)));
    CK(cudaMemset(ln.d_ld, 0, (P.T + 1) * sizeof(double)));
    if (P.R > 0) {
        CK(cudaMalloc(&ln.d_scratch, (size_t)P.R * P.nt * P.nt * sizeof(double)));
        CK(cudaMemset(ln.d_scratch, 0, (size_t)P.R * P.nt * P.nt * sizeof(double)));
    }
    return TC_OK;
}

int prep_all(tc_plan& P) {
    int r = prep_kernel((const void*)P.upd.fn, P.upd.smem);
    if (!r && P.upd_small.fn) r = prep_kernel((const void*)P.upd_small.fn, P.upd_small.smem);
    if (r) return r;
    bool in_smem;
    r = prep_kernel((const void*)k_potrf, (int)potrf_smem(P.nt, &in_smem));
    if (r) return r;
    const TrsmK TK = trsm_direct(P.nt);
    return prep_kernel((const void*)TK.fn, (int)TK.smem);
}

int build_graph(tc_plan& P, Lane& ln) {
    if (ln.exec) return TC_OK;
    int r = prep_all(P);
    if (r) return r;
    CK(cudaGraphCreate(&ln.graph, 0));
    std::vector<cudaGraphNode_t> nodes(P.launches.size());
    std::vector<cudaGraphNode_t> deps;
    for (size_t i = 0; i < P.launches.size(); ++i) {
        cudaKernelNodeParams kp;
        NodeArgs na;
        void* argv[8];
        r = node_params(P, ln, i, kp, na, argv);
        if (r) return r;
        deps.clear();
        for (int32_t d : P.launches[i].deps) deps.push_back(nodes[d]);
        CK(cudaGraphAddKernelNode(&nodes[i], ln.graph, deps.data(), deps.size(), &kp));
        cudaLaunchAttributeValue v;
        memset(&v, 0, sizeof v);
        v.priority = P.launches[i].high ? P.prio_hi : P.prio_lo;
        CK(cudaGraphKernelNodeSetAttribute(nodes[i], cudaLaunchAttributePriority, &v));
    }
    CK(cudaGraphInstantiateWithFlags(&ln.exec, ln.graph, cudaGraphInstantiateFlagUseNodePriority));
    return TC_OK;
}

int run_direct(tc_plan& P, Lane& ln, cudaStream_t s) {
    int r = prep_all(P);
    if (r) return r;
    for (size_t i = 0; i < P.launches.size(); ++i) {
        cudaKernelNodeParams kp;
        NodeArgs na;
        void* argv[8];
        r = node_params(P, ln, i, kp, na, argv);
        if (r) return r;
        CK(cudaLaunchKernel(kp.func, kp.gridDim, kp.blockDim, kp.kernelParams, kp.sharedMemBytes, s));
    }
    return TC_OK;
}

}  // namespace

extern "C" int tc_plan_create(int64_t n, int32_t nt, int64_t S, const int32_t* f_rows, const int32_t* f_cols,
                              const tc_plan_opts* opts, tc_plan_t* out) {
    if (!out || n < 1 || nt < 1 || S < 1 || !f_rows || !f_cols) return set_err(TC_ERR_ARG, "plan_create: bad arguments");
    *out = nullptr;
    if (tc_device_count() < 1) return set_err(TC_ERR_CUDA, "plan_create: no CUDA device");
    if (!potrf_supported(nt) || nt > kMaxTrsmNt)
        return set_err(TC_ERR_ARG, "plan_create: tile size %d unsupported (need nt<=160 or nt%%8==0, nt<=%d)", nt,
                       kMaxTrsmNt);
    std::unique_ptr<tc_plan> P(new tc_plan());
    P->n = n;
    P->nt = nt;
    P->T = (int)((n + nt - 1) / nt);
    P->S = S;
    if (opts) P->opts = *opts;
    else {
        memset(&P->opts, 0, sizeof P->opts);
        P->opts.lookahead = 1;
        P->opts.use_graph = 2;
    }
    P->W = P->opts.tree_workers > 0 ? P->opts.tree_workers : 8;
    P->fuse = P->opts.reserved[0] == 0 && !getenv("TC_NO_FUSE_TRSM");  // reserved[0] = 1 disables POTRF->TRSM streaming
    if (P->W > kMaxW) return set_err(TC_ERR_ARG, "plan_create: tree_workers <= %d", kMaxW);
    // The reference rule (chain >= 2 * workers) is sized for CPU threads; on
    // the device a chain only needs splitting when it is much longer than a
    // column step's K (the arrow x arrow chains of length ~T), so the default
    // threshold is 8 * W; 2 * W is available explicitly.
    if (P->opts.tree_threshold == 0) P->opts.tree_threshold = 8 * P->W;
    P->frow.assign(f_rows, f_rows + S);
    P->fcol.assign(f_cols, f_cols + S);
    P->upd = pick_upd(nt);
    P->upd_small = pick_upd_small(nt);
    CK(cudaGetDevice(&P->dev));
    CK(cudaDeviceGetStreamPriorityRange(&P->prio_lo, &P->prio_hi));
    int r = build_plan(*P);
    if (r) {
        tc_plan_destroy(P.release());
        return r;
    }
    *out = P.release();
    return TC_OK;
}

extern "C" int tc_plan_info(tc_plan_t p, int64_t* n_launches, int64_t* n_items, int64_t* n_pairs,
                            int64_t* scratch_tiles, double* tile_flops) {
    if (!p) return set_err(TC_ERR_ARG, "plan_info: null plan");
    if (n_launches) *n_launches = (int64_t)p->launches.size();
    if (n_items) *n_items = (int64_t)p->items.size();
    if (n_pairs) *n_pairs = (int64_t)p->pairs.size();
    if (scratch_tiles) *scratch_tiles = p->R;
    if (tile_flops) *tile_flops = p->flops;
    return TC_OK;
}

extern "C" int tc_plan_factorize_async(tc_plan_t p, int32_t lane, double* storage, void* stream) {
    if (!p || !storage) return set_err(TC_ERR_ARG, "plan_factorize: bad arguments");
    int r = ensure_lane(*p, lane);
    if (r) return r;
    Lane& ln = p->lanes[lane];
    cudaStream_t s = (cudaStream_t)stream;
    ln.h.storage = storage;
    ln.h.scratch = ln.d_scratch;
    ln.h.S = p->S;
    ln.h.fail = ln.d_fail;
    ln.h.ld_part = ln.d_ld;
    ln.h.ld_out = ln.d_ld + p->T;
    const int64_t nf = kNoFail;
    // context + failure word set by a 1-thread kernel: the values travel as
    // launch parameters (no pageable host source whose lifetime or staging
    // semantics could race with the lane's next call)
    k_set_ctx<<<1, 1, 0, s>>>(ln.d_ctx, ln.h, ln.d_fail, nf);
    CK(cudaGetLastError());
    if (p->opts.use_graph == 2) {
        r = run_persistent(*p, ln, s);
        if (r) return r;
    } else if (p->opts.use_graph) {
        r = build_graph(*p, ln);
        if (r) return r;
        CK(cudaGraphLaunch(ln.exec, s));
    } else {
        r = run_direct(*p, ln, s);
        if (r) return r;
    }
    return TC_OK;
}

extern "C" int tc_plan_collect(tc_plan_t p, int32_t lane, void* stream, int64_t* fail_index, double* logdet) {
    if (!p || lane < 0 || lane >= (int)p->lanes.size() || !p->lanes[lane].d_ctx)
        return set_err(TC_ERR_ARG, "plan_collect: bad lane");
    Lane& ln = p->lanes[lane];
    cudaStream_t s = (cudaStream_t)stream;
    int64_t f = kNoFail;
    double ld = 0.0;
    CK(cudaMemcpyAsync(&f, ln.d_fail, 8, cudaMemcpyDeviceToHost, s));
    CK(cudaMemcpyAsync(&ld, ln.d_ld + p->T, 8, cudaMemcpyDeviceToHost, s));
    CK(cudaStreamSynchronize(s));
    if (fail_index) *fail_index = (f == kNoFail) ? -1 : f;
    if (logdet) *logdet = ld;
    return TC_OK;
}

// Debug: current ticket of a lane's running persistent kernel (copied on a
// private non-blocking stream, so it can be read while the kernel spins).
extern "C" int tc_plan_debug_ticket(tc_plan_t p, int32_t lane, int32_t* ticket, int32_t* ntasks) {
    if (!p || lane < 0 || lane >= (int)p->lanes.size() || !p->lanes[lane].d_pstate)
        return set_err(TC_ERR_ARG, "plan_debug_ticket: bad lane");
    cudaStream_t s;
    CK(cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking));
    const size_t NL = p->launches.size();
    CK(cudaMemcpyAsync(ticket, p->lanes[lane].d_pstate + 2 * NL, 4, cudaMemcpyDeviceToHost, s));
    if (getenv("TC_DEBUG_DUMP")) {  // remaining/deps + ticket order of every launch -> file
        std::vector<int32_t> st(2 * NL);
        CK(cudaMemcpyAsync(st.data(), p->lanes[lane].d_pstate, 2 * NL * 4, cudaMemcpyDeviceToHost, s));
        CK(cudaStreamSynchronize(s));
        char fn[512];
        snprintf(fn, sizeof fn, "%s.%d", getenv("TC_DEBUG_DUMP"), lane);
        FILE* f = fopen(fn, "w");
        std::vector<int64_t> first(NL, -1);
        for (size_t t = 0; t < p->ptasks.size(); ++t)
            if (first[p->ptasks[t].launch] < 0) first[p->ptasks[t].launch] = (int64_t)t;
        for (size_t i = 0; i < NL; ++i)
            fprintf(f, "%zu %d %d %d %d %lld\n", i, p->launches[i].kind, p->launches[i].k, st[i], st[NL + i],
                    (long long)first[i]);
        fclose(f);
        std::vector<int32_t> pr(p->T, -7);
        int64_t fw = 0;
        if (p->lanes[lane].d_prog)
            CK(cudaMemcpyAsync(pr.data(), p->lanes[lane].d_prog, p->T * 4, cudaMemcpyDeviceToHost, s));
        CK(cudaMemcpyAsync(&fw, p->lanes[lane].d_fail, 8, cudaMemcpyDeviceToHost, s));
        CK(cudaStreamSynchronize(s));
        snprintf(fn, sizeof fn, "%s.%d.prog", getenv("TC_DEBUG_DUMP"), lane);
        f = fopen(fn, "w");
        fprintf(f, "fail %lld\n", (long long)fw);
        for (int k = 0; k < p->T; ++k) fprintf(f, "%d %d\n", k, pr[k]);
        fclose(f);
    }
    CK(cudaStreamSynchronize(s));
    cudaStreamDestroy(s);
    *ntasks = (int32_t)p->ptasks.size();
    return TC_OK;
}

// Asynchronous result hand-off for streaming batches: enqueue device-to-device
// copies of a lane's failure word (kNoFail = INT64_MAX when the factorisation
// succeeded) and log-determinant into caller buffers, so the lane can take the
// next problem without a host round trip.
extern "C" int tc_plan_copy_result(tc_plan_t p, int32_t lane, void* stream, int64_t* fail_dev, double* logdet_dev) {
    if (!p || lane < 0 || lane >= (int)p->lanes.size() || !p->lanes[lane].d_ctx)
        return set_err(TC_ERR_ARG, "plan_copy_result: bad lane");
    Lane& ln = p->lanes[lane];
    cudaStream_t s = (cudaStream_t)stream;
    if (fail_dev) CK(cudaMemcpyAsync(fail_dev, ln.d_fail, 8, cudaMemcpyDeviceToDevice, s));
    if (logdet_dev) CK(cudaMemcpyAsync(logdet_dev, ln.d_ld + p->T, 8, cudaMemcpyDeviceToDevice, s));
    return TC_OK;
}

extern "C" int tc_plan_factorize(tc_plan_t p, double* storage, void* stream, int64_t* fail_index) {
    int r = tc_plan_factorize_async(p, 0, storage, stream);
    if (r) return r;
    return tc_plan_collect(p, 0, stream, fail_index, nullptr);
}

extern "C" int tc_plan_logdet(tc_plan_t p, const double* storage, void* stream, double* out) {
    if (!p || !storage || !out) return set_err(TC_ERR_ARG, "plan_logdet: bad arguments");
    cudaStream_t s = (cudaStream_t)stream;
    double* part = nullptr;
    CK(cudaMallocAsync((void**)&part, (p->T + 1) * sizeof(double), s));
    k_logdet_tiles<<<p->T, 32, 0, s>>>(storage, p->d_diag_slots, p->T, p->nt, p->n, part);
    k_sum_fixed<<<1, 256, 0, s>>>(part, p->T, 2.0, part + p->T);
    CK(cudaGetLastError());
    CK(cudaMemcpyAsync(out, part + p->T, 8, cudaMemcpyDeviceToHost, s));
    cudaFreeAsync(part, s);
    CK(cudaStreamSynchronize(s));
    return TC_OK;
}

extern "C" int tc_plan_solve(tc_plan_t p, const double* storage, double* rhs, int32_t nrhs, void* stream) {
    if (!p || !storage || !rhs || nrhs < 1) return set_err(TC_ERR_ARG, "plan_solve: bad arguments");
    if (p->nt > kMaxTrsmNt) return set_err(TC_ERR_ARG, "plan_solve: nt > %d unsupported", kMaxTrsmNt);
    cudaStream_t s = (cudaStream_t)stream;
    const int nt = p->nt, T = p->T;
    const int64_t ldr = (int64_t)T * nt;
    const size_t nt2 = (size_t)nt * nt;
    // (1) Winv_k = L_kk^-T for every diagonal tile: batched TRSM of the identity
    double* W = nullptr;
    int32_t* flags = nullptr;
    CK(cudaMallocAsync((void**)&W, nt2 * T * sizeof(double), s));
    CK(cudaMallocAsync((void**)&flags, (2 * (size_t)T + 1) * sizeof(int32_t), s));
    k_set_identity<<<592, 256, 0, s>>>(W, T, nt);
    int r = TC_OK;
    {
        const TrsmK TK = trsm_direct(nt);
        const size_t sm = TK.smem;
        r = prep_kernel((const void*)TK.fn, (int)sm);
        if (!r) {
            TrsmArgs ta{};
            ta.storage = const_cast<double*>(storage);
            ta.lslots = p->d_diag_slots;
            ta.X = W;
            ta.nt = nt;
            for (int k0 = 0; k0 < T && !r; k0 += 65535) {
                ta.lslots = p->d_diag_slots + k0;
                ta.X = W + (size_t)k0 * nt2;
                dim3 grid((nt + TK.rows - 1) / TK.rows, (unsigned)std::min(T - k0, 65535));
                TK.fn<<<grid, 4 * TK.rows, sm, s>>>(ta);
                cudaError_t e = cudaGetLastError();
                if (e != cudaSuccess) r = set_err(TC_ERR_CUDA, "solve trsm: %s", cudaGetErrorString(e));
            }
        }
    }
    // (2) both sweeps in one persistent launch, nrhs in chunks of kSolveMaxRhs
    if (!r) {
        const int rows = (nt + 31) & ~31;
        const int P = rows >= kSolveThreads ? 1 : kSolveThreads / rows;
        const size_t sm = ((size_t)2 * kSolveMaxRhs * nt + (size_t)P * kSolveMaxRhs * rows) * sizeof(double);
        r = prep_kernel((const void*)k_solve_sweep, (int)sm);
        int sms = 148;
        cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, p->dev);
        for (int c0 = 0; c0 < nrhs && !r; c0 += kSolveMaxRhs) {
            CK(cudaMemsetAsync(flags, 0, (2 * (size_t)T + 1) * sizeof(int32_t), s));
            SolveArgs sa{};
            sa.storage = storage;
            sa.winv = W;
            sa.rhs = rhs + (size_t)c0 * ldr;
            sa.ldr = ldr;
            sa.nt = nt;
            sa.T = T;
            sa.nrhs = std::min(kSolveMaxRhs, nrhs - c0);
            sa.row_ptr = p->d_row_ptr;
            sa.row_col = p->d_row_col;
            sa.row_slot = p->d_row_slot;
            sa.col_ptr = p->d_sol_off;
            sa.col_row = p->d_sol_rows;
            sa.col_slot = p->d_sol_slots;
            sa.done = flags;
            sa.ticket = flags + 2 * T;
            const int grid = std::max(1, std::min(2 * T, sms));
            k_solve_sweep<<<grid, kSolveThreads, sm, s>>>(sa);
            cudaError_t e = cudaGetLastError();
            if (e != cudaSuccess) r = set_err(TC_ERR_CUDA, "solve sweep: %s", cudaGetErrorString(e));
        }
    }
    cudaFreeAsync(W, s);
    cudaFreeAsync(flags, s);
    if (r) return r;
    return TC_OK;
}

extern "C" int tc_plan_pack_offsets(tc_plan_t p, int64_t n, const int64_t* col_ptr, const int32_t* row_idx,
                                    int64_t* offs) {
    if (!p || n != p->n || !col_ptr || !row_idx || !offs) return set_err(TC_ERR_ARG, "pack_offsets: bad arguments");
    const int nt = p->nt;
    const int64_t nt2 = (int64_t)nt * nt;
    for (int64_t c = 0; c < n; ++c) {
        const int32_t tc = (int32_t)(c / nt);
        int64_t s = p->cs[tc];
        const int64_t se = p->cs[tc + 1];
        for (int64_t e = col_ptr[c]; e < col_ptr[c + 1]; ++e) {
            const int32_t r = row_idx[e];
            if (r < c || r >= n) return set_err(TC_ERR_FORMAT, "pack_offsets: entry outside the lower triangle");
            const int32_t tr = r / nt;
            while (s < se && p->frow[s] < tr) ++s;
            if (s >= se || p->frow[s] != tr) {
                // rows are sorted within a column, but allow unsorted input via search
                const int64_t f = find_slot(*p, tr, tc);
                if (f < 0) return set_err(TC_ERR_ARG, "grid does not cover the matrix pattern");
                offs[e] = f * nt2 + (c % nt) * nt + (r % nt);
                s = p->cs[tc];
                continue;
            }
            offs[e] = s * nt2 + (c % nt) * nt + (r % nt);
        }
    }
    return TC_OK;
}

extern "C" int tc_plan_pack_lincomb(tc_plan_t p, const double* basis, int32_t nbasis, const double* coef,
                                    const int64_t* offs, int64_t nnz, double* storage, void* stream) {
    if (!p || !storage || !coef || nbasis < 1 || nbasis > kMaxBasis || (nnz > 0 && (!basis || !offs)))
        return set_err(TC_ERR_ARG, "plan_pack_lincomb: bad arguments (1 <= nbasis <= %d)", kMaxBasis);
    cudaStream_t s = (cudaStream_t)stream;
    const size_t bytes = (size_t)p->S * p->nt * p->nt * sizeof(double);
    CK(cudaMemsetAsync(storage, 0, bytes, s));
    if (nnz > 0) {
        Lincomb lc{};
        lc.m = nbasis;
        for (int i = 0; i < nbasis; ++i) lc.c[i] = coef[i];
        const int64_t blocks = std::min<int64_t>((nnz + 255) / 256, 148 * 16);
        k_pack_lincomb<<<(unsigned)blocks, 256, 0, s>>>(basis, nnz, lc, offs, storage);
    }
    const int from = (int)(p->n % p->nt);
    if (from) k_pad_diag<<<1, p->nt, 0, s>>>(storage, p->cs[p->T - 1], p->nt, from);
    CK(cudaGetLastError());
    return TC_OK;
}

extern "C" int tc_plan_pack(tc_plan_t p, const double* vals, const int64_t* offs, int64_t nnz, double* storage,
                            void* stream) {
    if (!p || !storage || (nnz > 0 && (!vals || !offs))) return set_err(TC_ERR_ARG, "plan_pack: bad arguments");
    cudaStream_t s = (cudaStream_t)stream;
    const size_t bytes = (size_t)p->S * p->nt * p->nt * sizeof(double);
    CK(cudaMemsetAsync(storage, 0, bytes, s));
    if (nnz > 0) {
        const int64_t blocks = std::min<int64_t>((nnz + 255) / 256, 148 * 16);
        k_pack<<<(unsigned)blocks, 256, 0, s>>>(vals, offs, nnz, storage);
    }
    const int from = (int)(p->n % p->nt);
    if (from) k_pad_diag<<<1, p->nt, 0, s>>>(storage, p->cs[p->T - 1], p->nt, from);
    CK(cudaGetLastError());
    return TC_OK;
}

extern "C" void tc_plan_destroy(tc_plan_t p) {
    if (!p) return;
    for (auto& ln : p->lanes) {
        if (ln.exec) cudaGraphExecDestroy(ln.exec);
        if (ln.graph) cudaGraphDestroy(ln.graph);
        cudaFree(ln.d_ctx);
        cudaFree(ln.d_fail);
        cudaFree(ln.d_ld);
        cudaFree(ln.d_scratch);
        cudaFree(ln.d_pstate);
        cudaFree(ln.d_prog);
        cudaFree(ln.d_xctr);
    }
    cudaFree(p->d_ptasks);
    cudaFree(p->d_plaunch);
    cudaFree(p->d_p_init);
    cudaFree(p->d_succ_ptr);
    cudaFree(p->d_succ);
    cudaFree(p->d_xctr_of_slot);
    cudaFree(p->d_items);
    cudaFree(p->d_pairs);
    cudaFree(p->d_tgts);
    cudaFree(p->d_diag_slots);
    cudaFree(p->d_sol_slots);
    cudaFree(p->d_sol_rows);
    cudaFree(p->d_sol_off);
    cudaFree(p->d_row_ptr);
    cudaFree(p->d_row_col);
    cudaFree(p->d_row_slot);
    delete p;
}

// Host staging for the end-to-end path: page-lock a caller's host array in
// place (no copy) so its per-call H2D runs at pinned bandwidth, and an async
// copy that does not depend on the caller knowing the pointer is registered.
extern "C" int tc_host_register(void* ptr, size_t bytes) {
    if (!ptr || !bytes) return set_err(TC_ERR_ARG, "host_register: bad arguments");
    const cudaError_t e = cudaHostRegister(ptr, bytes, cudaHostRegisterDefault);
    if (e != cudaSuccess) {
        // already registered / read-only mapping / overlapping range: the
        // caller falls back to a staging copy; clear the sticky last-error
        // slot so a later CK(cudaGetLastError()) does not report it
        cudaGetLastError();
        return set_err(TC_ERR_CUDA, "cudaHostRegister: %s", cudaGetErrorString(e));
    }
    return TC_OK;
}
extern "C" int tc_host_unregister(void* ptr) {
    if (!ptr) return set_err(TC_ERR_ARG, "host_unregister: null");
    const cudaError_t e = cudaHostUnregister(ptr);
    if (e != cudaSuccess) {
        cudaGetLastError();
        return set_err(TC_ERR_CUDA, "cudaHostUnregister: %s", cudaGetErrorString(e));
    }
    return TC_OK;
}
extern "C" int tc_memcpy_h2d_async(void* dst_dev, const void* src_host, size_t bytes, void* stream) {
    if (!dst_dev || !src_host) return set_err(TC_ERR_ARG, "memcpy_h2d_async: bad arguments");
    CK(cudaMemcpyAsync(dst_dev, src_host, bytes, cudaMemcpyHostToDevice, (cudaStream_t)stream));
    return TC_OK;
}

// error hook shared with the host-analysis translation unit (tc_host.cpp)
extern "C" int tc__set_error(int code, const char* msg) {
    g_err = msg;
    return code;
}

// ---------------------------------------------------------------- profiling --
// Serialised pass of the plan on one stream with CUDA events around every
// launch; per profiling class: total ms, launch count, algorithmic flops.
extern "C" int tc_plan_profile(tc_plan_t p, double* storage, void* stream, int32_t n_cls, double* ms,
                               int64_t* counts, double* flops) {
    if (!p || !storage || n_cls < 7 || !ms || !counts || !flops) return set_err(TC_ERR_ARG, "plan_profile: bad arguments");
    int r = ensure_lane(*p, 0);
    if (r) return r;
    r = prep_all(*p);
    if (r) return r;
    Lane& ln = p->lanes[0];
    cudaStream_t s = (cudaStream_t)stream;
    ln.h.storage = storage;
    ln.h.scratch = ln.d_scratch;
    ln.h.S = p->S;
    ln.h.fail = ln.d_fail;
    ln.h.ld_part = ln.d_ld;
    ln.h.ld_out = ln.d_ld + p->T;
    const int64_t nf = kNoFail;
    // context + failure word set by a 1-thread kernel: the values travel as
    // launch parameters (no pageable host source whose lifetime or staging
    // semantics could race with the lane's next call)
    k_set_ctx<<<1, 1, 0, s>>>(ln.d_ctx, ln.h, ln.d_fail, nf);
    CK(cudaGetLastError());
    const size_t NL = p->launches.size();
    std::vector<cudaEvent_t> ev(NL + 1);
    for (auto& e : ev) CK(cudaEventCreate(&e));
    CK(cudaEventRecord(ev[0], s));
    for (size_t i = 0; i < NL; ++i) {
        cudaKernelNodeParams kp;
        NodeArgs na;
        void* argv[8];
        r = node_params(*p, ln, i, kp, na, argv);
        if (r) return r;
        CK(cudaLaunchKernel(kp.func, kp.gridDim, kp.blockDim, kp.kernelParams, kp.sharedMemBytes, s));
        CK(cudaEventRecord(ev[i + 1], s));
    }
    CK(cudaStreamSynchronize(s));
    for (int c = 0; c < n_cls; ++c) {
        ms[c] = 0.0;
        counts[c] = 0;
        flops[c] = 0.0;
    }
    for (size_t i = 0; i < NL; ++i) {
        float t = 0.f;
        CK(cudaEventElapsedTime(&t, ev[i], ev[i + 1]));
        const int c = p->launches[i].cls;
        ms[c] += t;
        counts[c] += 1;
        flops[c] += p->launches[i].flops;
    }
    for (auto& e : ev) cudaEventDestroy(e);
    return TC_OK;
}

// Task trace of one persistent-executor factorisation: per task (ticket
// order) the ns timestamps when its CTA took the ticket, when the task's
// launch became runnable and when the task finished, and the SM id; per
// launch its kind (0 update, 1 POTRF, 2 TRSM, 3 combine, 4 logdet), column
// and profiling class.  Factorises storage_dev in place.
extern "C" int tc_plan_trace(tc_plan_t p, double* storage, void* stream, int64_t cap, int64_t* tasks_out,
                             int32_t* task_launch, int64_t launch_cap, int32_t* launch_meta, int64_t* n_tasks,
                             int64_t* n_launches) {
    if (!p || !storage || !n_tasks || !n_launches) return set_err(TC_ERR_ARG, "plan_trace: bad arguments");
    if (p->opts.use_graph != 2) return set_err(TC_ERR_ARG, "plan_trace: persistent executor only");
    const int64_t NT = (int64_t)p->ptasks.size(), NL = (int64_t)p->launches.size();
    *n_tasks = NT;
    *n_launches = NL;
    if (cap < NT || launch_cap < NL || !tasks_out || !task_launch || !launch_meta) return TC_OK;  // size query
    int r = ensure_lane(*p, 0);
    if (r) return r;
    Lane& ln = p->lanes[0];
    cudaStream_t s = (cudaStream_t)stream;
    CK(cudaMalloc(&ln.d_trace, (size_t)NT * 4 * sizeof(int64_t)));
    CK(cudaMemsetAsync(ln.d_trace, 0, (size_t)NT * 4 * sizeof(int64_t), s));
    r = tc_plan_factorize_async(p, 0, storage, stream);
    if (!r) CK(cudaMemcpyAsync(tasks_out, ln.d_trace, (size_t)NT * 4 * sizeof(int64_t), cudaMemcpyDeviceToHost, s));
    CK(cudaStreamSynchronize(s));
    cudaFree(ln.d_trace);
    ln.d_trace = nullptr;
    if (r) return r;
    for (int64_t t = 0; t < NT; ++t) task_launch[t] = p->ptasks[t].launch;
    for (int64_t i = 0; i < NL; ++i) {
        launch_meta[3 * i] = p->launches[i].kind | p->launches[i].tag;
        launch_meta[3 * i + 1] = p->launches[i].k;
        launch_meta[3 * i + 2] = p->launches[i].cls;
    }
    return TC_OK;
}

// DMMA throughput microbenchmark: every warp issues independent m8n8k4 FP64
// MMAs from registers; returns TFLOP/s over the whole device.
namespace {
__global__ void k_dmma_peak(int64_t iters, double* sink) {
    double a = threadIdx.x * 1e-3, b = blockIdx.x * 1e-3;
    double d[8][2];
#pragma unroll
    for (int i = 0; i < 8; ++i) d[i][0] = d[i][1] = 0.0;
    for (int64_t it = 0; it < iters; ++it) {
#pragma unroll
        for (int i = 0; i < 8; ++i) dmma(d[i][0], d[i][1], a, b);
    }
    double s = 0.0;
#pragma unroll
    for (int i = 0; i < 8; ++i) s += d[i][0] + d[i][1];
    if (s == 12345.678) sink[0] = s;
}
}  // namespace

extern "C" int tc_bench_dmma_peak(int64_t iters, int32_t blocks_per_sm, int32_t warps_per_block, double* tflops) {
    if (iters < 1 || !tflops) return set_err(TC_ERR_ARG, "dmma_peak: bad arguments");
    int dev = 0, sms = 0;
    CK(cudaGetDevice(&dev));
    CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
    double* sink = nullptr;
    CK(cudaMalloc(&sink, 8));
    const int grid = sms * blocks_per_sm, block = 32 * warps_per_block;
    k_dmma_peak<<<grid, block>>>(iters / 10 + 1, sink);
    cudaEvent_t a, b;
    CK(cudaEventCreate(&a));
    CK(cudaEventCreate(&b));
    CK(cudaEventRecord(a));
    k_dmma_peak<<<grid, block>>>(iters, sink);
    CK(cudaEventRecord(b));
    CK(cudaEventSynchronize(b));
    float ms = 0.f;
    CK(cudaEventElapsedTime(&ms, a, b));
    const double fl = 2.0 * 256.0 * 8.0 * (double)iters * grid * warps_per_block;  // 256 FMA per DMMA per warp
    *tflops = fl / (ms * 1e-3) / 1e12;
    cudaFree(sink);
    cudaEventDestroy(a);
    cudaEventDestroy(b);
    return TC_OK;
}
