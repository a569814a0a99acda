// Standalone GEMM entry used by the parity tests of the tensor-core kernel
// itself (tests/test_gpu_gemm.py): plain store epilogue, every majorness /
// dtype / tile-width combination the layer kernels instantiate.
#include <cstring>

#include "../../include/cdp_b200.h"
#include "gemm_launch.cuh"

namespace cdp {

struct EpiStore {
    struct Params {
        float *d;
        int ldd;
    };
    static constexpr bool kTile = false;
    static constexpr int kStages = 0;
    template <int BN>
    static constexpr int pf_bytes() { return 0; }
    template <int BN>
    __device__ static void prefetch(const Params &, float *, int, int, int, int, int, int) {}
    struct State {};
    template <int BN>
    __device__ static void tile(const Params &, const float *, int, const float *, int, int, int, int, int, int) {}
    __device__ static void begin(const Params &, int, State &) {}
    __device__ static void finish(const Params &, int, int, State &) {}
    __device__ static void apply(const Params &p, int m, int n0, const float (&v)[32], int M, int N, State &) {
        if (m >= M) return;
#pragma unroll
        for (int i = 0; i < 32; ++i)
            if (n0 + i < N) p.d[size_t(m) * p.ldd + n0 + i] = v[i];
    }
    __device__ static void extra(const Params &, int, int) {}
    __device__ static void pre(const Params &, int) {}
    __device__ static void post(const Params &, int, unsigned) {}
};

template <int KIND, int BN, bool A_MN, bool B_MN>
static void run_test(const Operand *A, const Operand *B, int n_seg, int M, int N, int K, float *D, int ldd,
                     int splits, float *ws, int *counters, cudaStream_t st) {
    GemmPlan p = plan_gemm<KIND, BN, A_MN, B_MN>(A, B, n_seg, M, N, K, splits, ws, counters);
    launch_gemm<KIND, BN, A_MN, B_MN, EpiStore>(p, EpiStore::Params{D, ldd}, st);
}

template <int KIND, int BN>
static void dispatch_major(bool amn, bool bmn, const Operand *A, const Operand *B, int n_seg, int M, int N, int K,
                           float *D, int ldd, int splits, float *ws, int *counters, cudaStream_t st) {
    if (!amn && !bmn) run_test<KIND, BN, false, false>(A, B, n_seg, M, N, K, D, ldd, splits, ws, counters, st);
    if (amn && !bmn) run_test<KIND, BN, true, false>(A, B, n_seg, M, N, K, D, ldd, splits, ws, counters, st);
    if constexpr (BN % (KIND == 0 ? 64 : 32) == 0) {
        if (!amn && bmn) run_test<KIND, BN, false, true>(A, B, n_seg, M, N, K, D, ldd, splits, ws, counters, st);
        if (amn && bmn) run_test<KIND, BN, true, true>(A, B, n_seg, M, N, K, D, ldd, splits, ws, counters, st);
    } else {
        if (bmn) throw CdpError("MN-major B needs BN multiple of 128 bytes");
    }
}

}  // namespace cdp

using namespace cdp;

extern "C" int cdp_test_gemm(int kind, int a_mn, int b_mn, int bn, int M, int N, int K, int n_seg,
                             const void *const *a_ptrs, int lda, const void *const *b_ptrs, int ldb, float *d, int ldd,
                             int splits, float *ws, int *counters, void *stream) {
    return guarded([&] {
        Operand A[3], B[3];
        for (int s = 0; s < n_seg; ++s) {
            A[s] = Operand{a_ptrs[s], a_mn != 0, uint64_t(M), uint64_t(K), uint64_t(lda)};
            B[s] = Operand{b_ptrs[s], b_mn != 0, uint64_t(N), uint64_t(K), uint64_t(ldb)};
        }
        cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
        const bool amn = a_mn, bmn = b_mn;
#define CDP_BN(K_, BN_) \
    if (kind == K_ && bn == BN_) { dispatch_major<K_, BN_>(amn, bmn, A, B, n_seg, M, N, K, d, ldd, splits, ws, counters, st); return; }
        CDP_BN(0, 32) CDP_BN(0, 64) CDP_BN(0, 128) CDP_BN(0, 256)
        CDP_BN(1, 32) CDP_BN(1, 64) CDP_BN(1, 128) CDP_BN(1, 256)
#undef CDP_BN
        throw CdpError("unsupported gemm test configuration");
    });
}
