// Layer kernels of the stage-stacked tanh MLP (ref training/_kernels.pyx:25-132)
// as fused epilogues of the tcgen05 GEMM, plus the loss and gather kernels.
//
// Compute formats (template KIND):
//   0  bf16 operands      : one bf16 array per tensor
//   1  fp32 as 3xTF32     : hi = x with the 13 low mantissa bits cleared (exact
//                           tf32), lo = x - hi (exact); products hi.hi+hi.lo+lo.hi
#pragma once
#include <cuda_bf16.h>

#include "gemm.cuh"

namespace cdp {

template <int KIND>
struct Fmt;

template <>
struct Fmt<0> {
    __device__ static void store(void *hi, void *, size_t i, float x) {
        static_cast<__nv_bfloat16 *>(hi)[i] = __float2bfloat16_rn(x);
    }
    __device__ static float load(const void *hi, const void *, size_t i) {
        return __bfloat162float(static_cast<const __nv_bfloat16 *>(hi)[i]);
    }
};

template <>
struct Fmt<1> {
    __device__ static void store(void *hi, void *lo, size_t i, float x) {
        const float h = __uint_as_float(__float_as_uint(x) & 0xFFFFE000u);
        static_cast<float *>(hi)[i] = h;
        static_cast<float *>(lo)[i] = __fsub_rn(x, h);
    }
    __device__ static float load(const void *hi, const void *lo, size_t i) {
        return __fadd_rn(static_cast<const float *>(hi)[i], static_cast<const float *>(lo)[i]);
    }
};

// Compute-format tensor: hi (and lo for KIND 1), row stride ld elements.
struct CTensor {
    void *hi;
    void *lo;
    int ld;
};

// ---------------------------------------------------------------------------
// Forward: accumulator = (W^T . H^T)[o, s].  out[s, o] = tanh(acc + b[o]) in
// compute format (next stage input), or z[s, o] = acc + b[o] in fp32 for the
// last stage (ref _kernels.pyx:40-62).
template <int KIND>
struct EpiFwd {
    // The stage input record carries a ones column at index din and the packed
    // weights a bias row at index din (the reference's flat stage layout
    // [din][dout] + [dout] IS the [din+1][dout] matrix), so acc already holds
    // h.W + b.
    struct Params {
        CTensor out;  // next-stage input record (tanh applied)
        float *z;     // last stage: fp32 logits [B][dout]
        int last;
    };
    struct State {};
    __device__ static void begin(const Params &, int, State &) {}
    __device__ static void apply(const Params &p, int m, int n0, const float (&v)[32], int M, int N, State &) {
        if (m >= M) return;
#pragma unroll 8
        for (int i = 0; i < 32; ++i) {
            const int s = n0 + i;
            if (s < N) {
                if (p.last)
                    p.z[size_t(s) * M + m] = v[i];
                else
                    Fmt<KIND>::store(p.out.hi, p.out.lo, size_t(s) * p.out.ld + m, tanhf(v[i]));
            }
        }
    }
    __device__ static void finish(const Params &, int, int, State &) {}
    __device__ static void extra(const Params &, int, int) {}
    static constexpr bool kTile = false;
    static constexpr int kStages = 0;
    template <int BN>
    static constexpr int pf_bytes() { return 0; }
    template <int BN>
    __device__ static void prefetch(const Params &, float *, int, int, int, int, int, int) {}
    template <int BN>
    __device__ static void tile(const Params &, const float *, int, const float *, int, int, int, int, int, int) {}
    __device__ static void pre(const Params &, int) {}
    __device__ static void post(const Params &, int, unsigned) {}
};

// ---------------------------------------------------------------------------
// Data gradient: accumulator = (W . dZ^T)[k, s].  dprev[s, k] = acc * (1 - h^2)
// with h the stage input record, and the bias gradient of the previous stage
// db[k] = sum_s dprev[s, k] in ascending s (ref _kernels.pyx:115-130).
template <int KIND>
struct EpiDgrad {
    // accumulator = (W . dZ^T)[k, s];  dprev[s, k] = acc * (1 - h^2)  (ref _kernels.pyx:120-130)
    struct Params {
        CTensor h;      // stage-j input record (tanh outputs of stage j-1)
        CTensor dprev;  // dZ_{j-1} out
    };
    struct State {};
    __device__ static void begin(const Params &, int, State &) {}
    __device__ static void apply(const Params &p, int m, int n0, const float (&v)[32], int M, int N, State &) {
        if (m >= M) return;
        float h[32];
#pragma unroll
        for (int i = 0; i < 32; ++i)  // all 32 loads in flight before any use
            h[i] = (n0 + i < N) ? Fmt<KIND>::load(p.h.hi, p.h.lo, size_t(n0 + i) * p.h.ld + m) : 0.f;
#pragma unroll
        for (int i = 0; i < 32; ++i) {
            const int s = n0 + i;
            if (s < N)
                Fmt<KIND>::store(p.dprev.hi, p.dprev.lo, size_t(s) * p.dprev.ld + m,
                                 __fmul_rn(v[i], __fsub_rn(1.f, __fmul_rn(h[i], h[i]))));
        }
    }
    __device__ static void finish(const Params &, int, int, State &) {}
    __device__ static void extra(const Params &, int, int) {}
    static constexpr bool kTile = false;
    static constexpr int kStages = 0;
    template <int BN>
    static constexpr int pf_bytes() { return 0; }
    template <int BN>
    __device__ static void prefetch(const Params &, float *, int, int, int, int, int, int) {}
    template <int BN>
    __device__ static void tile(const Params &, const float *, int, const float *, int, int, int, int, int, int) {}
    __device__ static void pre(const Params &, int) {}
    __device__ static void post(const Params &, int, unsigned) {}
};

// ---------------------------------------------------------------------------
// Weight gradient fused with the CDP gradient hop and, on the last hop, the
// SGD(+momentum, weight decay) update (ref engine.py:96-109, comm.py:37-67).
// accumulator = (H1^T . dZ)[k, o] with H1 = [H, 1]: rows k < din are dW[k, o],
// row din is the bias gradient sum_s dZ[s, o] — the whole stage's flat gradient
// in the reference layout, computed by the tensor core in one GEMM.
//   mode 0 first hop : S[idx] = g
//   mode 1 mid hop   : S[idx] = S_in[idx] + g      (S_in: previous worker's
//                      partial; a peer-GPU pointer when workers are GPUs)
//   mode 2 last hop  : G = S_in[idx] + g, update
//   mode 3 only      : G = g (N = 1), update
//   mode 4 grad only : out[idx] = g (operator-level value+grad)
// Update (fp32): momentum: v = m*v + (G/n + wd*th); th' = th - lr*v.
//                no momentum: th' = th - (lr/n)*G   (wd: th - lr*(G/n + wd*th)).
// The new parameters are also written as the packed compute-format copy the
// next GEMMs read.  Non-finite gradient / parameter -> flag bits.
// Cross-GPU ring state, one per rank inside its IPC-shared region (flags are
// step / version numbers, written with st.release.sys, read with ld.acquire.sys).
constexpr int kMaxStages = 256;  // ring flag slots: one per hop unit (layer / parameter tensor)
struct RingFlags {
    uint32_t ready[kMaxStages];      // this rank's partial S^j is complete for step `ready[j]`
    uint32_t consumed[kMaxStages];   // the next rank finished reading this rank's S^j of that step
    uint32_t updated[kMaxStages];    // updater: stage j holds version `updated[j]`
    uint32_t pulled[kMaxStages][2];  // updater: readers that pulled version v (slot v % 2)
    uint32_t zdone[kMaxStages];      // ZeRO-CDP: global use index of this rank's last finished use of a unit
    uint32_t zcopied[kMaxStages];    // ZeRO-CDP frames: use index of the successor that copied this rank's unit
    uint32_t vtag[2][kMaxStages];    // trace mode: version held by theta slot s of unit j (travels with the data)
    uint32_t fwd_have[kMaxStages];   // pull chain: newest version of unit j this reader holds (pulled)
    uint32_t fwd_pulled[kMaxStages][2];  // pull chain: version the next reader took from this reader's slot
    uint32_t err;                    // a spin-wait timed out (protocol failure)
    uint32_t pad[31];
};

struct DistSync {
    int enabled;
    int n_readers;            // ranks that pull parameters (world - 1)
    const int *step;          // device control block step t
    RingFlags *own;
    RingFlags *prev;          // rank - 1 (peer memory), null on rank 0
    unsigned *cta_counter;    // local, per stage: CTAs of this launch that finished
    int pre_external;         // the pre-hop waits ran in a preceding one-CTA kernel (hop_wait_kernel)
};

// A wait that is not satisfied within ~9 s (2^34 cycles) is a protocol failure (or a peer that
// died): record it and trap, so the kernel never goes on to read partial sums / parameter slots
// that are not ready (the launch fails loudly instead of silently corrupting training).
__device__ __forceinline__ void spin_ge(const uint32_t *f, uint32_t v, uint32_t *err) {
    const long long t0 = clock64();
    while (ptx::ld_acquire_sys(f) < v) {
        if (clock64() - t0 > (1ll << 34)) {
            atomicExch(err, 1u);
            __threadfence_system();
            __trap();
        }
        __nanosleep(64);
    }
}

struct HopParams {
    int mode;
    int stage;            // 1-based
    int64_t base;         // stage offset in the flat parameter vector
    int din, dout;
    const float *s_in;
    float *s_out;
    const float *theta_cur;
    float *theta_new;
    float *vel;
    const float *lr;      // device scalar (per-step learning rate)
    float momentum, wd, n_mb;
    CTensor wc_new;       // packed compute copy of [W; b] (new version)
    unsigned *grad_flags; // bit (stage-1): non-finite gradient
    unsigned *upd_flags;  // bit (stage-1): non-finite updated parameter
    DistSync sync;        // multi-GPU ring protocol (sync.enabled = 0 on one GPU)
};

template <int KIND>
__device__ __forceinline__ void store_wc4(const CTensor &t, size_t i, float4 v) {
    if constexpr (KIND == 0) {
        __nv_bfloat162 a = __floats2bfloat162_rn(v.x, v.y), b = __floats2bfloat162_rn(v.z, v.w);
        uint2 u;
        u.x = *reinterpret_cast<uint32_t *>(&a);
        u.y = *reinterpret_cast<uint32_t *>(&b);
        *reinterpret_cast<uint2 *>(static_cast<__nv_bfloat16 *>(t.hi) + i) = u;
    } else {
        float4 h;
        h.x = __uint_as_float(__float_as_uint(v.x) & 0xFFFFE000u);
        h.y = __uint_as_float(__float_as_uint(v.y) & 0xFFFFE000u);
        h.z = __uint_as_float(__float_as_uint(v.z) & 0xFFFFE000u);
        h.w = __uint_as_float(__float_as_uint(v.w) & 0xFFFFE000u);
        *reinterpret_cast<float4 *>(static_cast<float *>(t.hi) + i) = h;
        *reinterpret_cast<float4 *>(static_cast<float *>(t.lo) + i) =
            make_float4(__fsub_rn(v.x, h.x), __fsub_rn(v.y, h.y), __fsub_rn(v.z, h.z), __fsub_rn(v.w, h.w));
    }
}

// The update arithmetic of one element (mirrors ref engine.py:102-109 in fp32).
__device__ __forceinline__ float sgd_update(const HopParams &p, float G, float th, float &v, float lr) {
    if (p.momentum != 0.f) {
        float gg = __fdiv_rn(G, p.n_mb);
        if (p.wd != 0.f) gg = __fadd_rn(gg, __fmul_rn(p.wd, th));
        v = __fadd_rn(__fmul_rn(v, p.momentum), gg);
        return __fsub_rn(th, __fmul_rn(lr, v));
    }
    if (p.wd != 0.f) return __fsub_rn(th, __fmul_rn(lr, __fadd_rn(__fdiv_rn(G, p.n_mb), __fmul_rn(p.wd, th))));
    return __fsub_rn(th, __fmul_rn(__fdiv_rn(lr, p.n_mb), G));
}

template <int KIND>
__device__ __forceinline__ void hop_elem(const HopParams &p, int64_t idx, float g, size_t widx, bool is_w,
                                         bool &bad_g, bool &bad_u) {
    if (!isfinite(g)) bad_g = true;
    if (p.mode == 0 || p.mode == 4) {
        p.s_out[idx] = g;
        return;
    }
    if (p.mode == 1) {
        p.s_out[idx] = __fadd_rn(__ldcg(p.s_in + idx), g);
        return;
    }
    const float G = p.mode == 2 ? __fadd_rn(__ldcg(p.s_in + idx), g) : g;
    float v = p.momentum != 0.f ? p.vel[idx] : 0.f;
    const float nt = sgd_update(p, G, p.theta_cur[idx], v, *p.lr);
    if (p.momentum != 0.f) p.vel[idx] = v;
    if (!isfinite(nt)) bad_u = true;
    p.theta_new[idx] = nt;
    if (is_w) Fmt<KIND>::store(p.wc_new.hi, p.wc_new.lo, widx, nt);
}

__device__ __forceinline__ bool finite4(float4 a) {
    return isfinite(a.x) && isfinite(a.y) && isfinite(a.z) && isfinite(a.w);
}

template <int KIND>
struct EpiWgrad {
    using Params = HopParams;
    static constexpr bool kTile = true;
    static constexpr int kStages = 2;  // K = micro-batch: at most a few k-blocks
    // prefetch area: theta_cur, velocity, incoming partial; [3][128][BN] fp32
    template <int BN>
    static constexpr int pf_bytes() { return 3 * 128 * BN * 4; }
    __device__ static bool vec_ok(const Params &p) { return (p.dout % 4 == 0) && (p.base % 4 == 0); }

    // Issued by the 128 epilogue threads while TMA + MMA still run (cp.async,
    // no registers held): every 16-byte slot of the tile this CTA will update.
    template <int BN>
    __device__ static void prefetch(const Params &p, float *pf, int m0, int n0, int M, int N, int tid, int nth) {
        if (!vec_ok(p)) return;
        const bool need_th = p.mode == 2 || p.mode == 3;
        const bool need_v = need_th && p.momentum != 0.f;
        const bool need_s = p.mode == 1 || p.mode == 2;
        constexpr int C4 = BN / 4;
        for (int e = tid; e < 128 * C4; e += nth) {
            const int r = e / C4, c = (e % C4) * 4;
            const int m = m0 + r, n = n0 + c;
            if (m >= M || n >= N) continue;
            const int64_t idx = p.base + int64_t(m) * p.dout + n;
            const int so = r * BN + c;
            if (need_th) ptx::cp_async16(pf + so, p.theta_cur + idx);
            if (need_v) ptx::cp_async16(pf + 128 * BN + so, p.vel + idx);
            if (need_s) ptx::cp_async16(pf + 2 * 128 * BN + so, p.s_in + idx);
        }
    }
    struct State {};
    __device__ static void begin(const Params &, int, State &) {}
    __device__ static void apply(const Params &, int, int, const float (&)[32], int, int, State &) {}
    __device__ static void finish(const Params &, int, int, State &) {}

    // The 128 x BN tile of dW sits in shared memory (row-major, stride lds).
    // Threads sweep it in float4 slots so consecutive threads touch consecutive
    // 16-byte chunks of a parameter row; U slots per thread are loaded before
    // any is consumed (memory-level parallelism for the peer / HBM reads).
    template <int BN>
    __device__ static void tile(const Params &p, const float *st, int lds, const float *pf, int m0, int n0, int M,
                                int N, int tid, int nth) {
        bool bad_g = false, bad_u = false;
        if (vec_ok(p)) {
            constexpr int C4 = BN / 4;
            constexpr int U = 4;
            const float lr = *p.lr;
            const int total = 128 * C4;
            for (int e0 = tid; e0 < total; e0 += nth * U) {
                float4 g[U], s[U], th[U], vv[U];
                int64_t idx[U];
                size_t widx[U];
                bool ok[U];
#pragma unroll
                for (int u = 0; u < U; ++u) {
                    const int e = e0 + u * nth;
                    const int r = e / C4, c = (e % C4) * 4;
                    const int m = m0 + r, n = n0 + c;
                    ok[u] = e < total && m < M && n < N;
                    if (!ok[u]) continue;
                    idx[u] = p.base + int64_t(m) * p.dout + n;
                    widx[u] = size_t(m) * p.wc_new.ld + n;
                    g[u] = *reinterpret_cast<const float4 *>(st + r * lds + c);
                    if (pf) {
                        const int so = r * BN + c;  // prefetched operands (shared)
                        if (p.mode == 1 || p.mode == 2) s[u] = *reinterpret_cast<const float4 *>(pf + 2 * 128 * BN + so);
                        if (p.mode == 2 || p.mode == 3) {
                            th[u] = *reinterpret_cast<const float4 *>(pf + so);
                            if (p.momentum != 0.f) vv[u] = *reinterpret_cast<const float4 *>(pf + 128 * BN + so);
                        }
                    } else {  // split-K tail CTA: operands straight from global memory
                        if (p.mode == 1 || p.mode == 2) s[u] = __ldcg(reinterpret_cast<const float4 *>(p.s_in + idx[u]));
                        if (p.mode == 2 || p.mode == 3) {
                            th[u] = *reinterpret_cast<const float4 *>(p.theta_cur + idx[u]);
                            if (p.momentum != 0.f) vv[u] = *reinterpret_cast<const float4 *>(p.vel + idx[u]);
                        }
                    }
                }
#pragma unroll
                for (int u = 0; u < U; ++u) {
                    if (!ok[u]) continue;
                    if (!finite4(g[u])) bad_g = true;
                    float4 *so = reinterpret_cast<float4 *>(p.s_out + idx[u]);
                    if (p.mode == 0 || p.mode == 4) {
                        *so = g[u];
                        continue;
                    }
                    float4 G = g[u];
                    if (p.mode == 1 || p.mode == 2)
                        G = make_float4(__fadd_rn(s[u].x, g[u].x), __fadd_rn(s[u].y, g[u].y),
                                        __fadd_rn(s[u].z, g[u].z), __fadd_rn(s[u].w, g[u].w));
                    if (p.mode == 1) {
                        *so = G;
                        continue;
                    }
                    float4 v = p.momentum != 0.f ? vv[u] : make_float4(0.f, 0.f, 0.f, 0.f);
                    float4 nt;
                    nt.x = sgd_update(p, G.x, th[u].x, v.x, lr);
                    nt.y = sgd_update(p, G.y, th[u].y, v.y, lr);
                    nt.z = sgd_update(p, G.z, th[u].z, v.z, lr);
                    nt.w = sgd_update(p, G.w, th[u].w, v.w, lr);
                    if (p.momentum != 0.f) *reinterpret_cast<float4 *>(p.vel + idx[u]) = v;
                    if (!finite4(nt)) bad_u = true;
                    *reinterpret_cast<float4 *>(p.theta_new + idx[u]) = nt;
                    store_wc4<KIND>(p.wc_new, widx[u], nt);
                }
            }
        } else {
            // unaligned rows (e.g. dout = 10): scalar, but only valid elements and
            // with U independent loads in flight per thread
            const int rows = min(128, M - m0), cols = min(BN, N - n0);
            const int total = rows * cols;
            constexpr int U = 8;
            const float lr = *p.lr;
            for (int e0 = tid; e0 < total; e0 += nth * U) {
                float g[U], sv[U], th[U], vv[U];
                int64_t idx[U];
                size_t widx[U];
                bool ok[U];
#pragma unroll
                for (int u = 0; u < U; ++u) {
                    const int e = e0 + u * nth;
                    ok[u] = e < total;
                    if (!ok[u]) continue;
                    const int r = e / cols, c = e % cols;
                    idx[u] = p.base + int64_t(m0 + r) * p.dout + n0 + c;
                    widx[u] = size_t(m0 + r) * p.wc_new.ld + n0 + c;
                    g[u] = st[r * lds + c];
                    if (p.mode == 1 || p.mode == 2) sv[u] = __ldcg(p.s_in + idx[u]);
                    if (p.mode == 2 || p.mode == 3) {
                        th[u] = p.theta_cur[idx[u]];
                        if (p.momentum != 0.f) vv[u] = p.vel[idx[u]];
                    }
                }
#pragma unroll
                for (int u = 0; u < U; ++u) {
                    if (!ok[u]) continue;
                    if (!isfinite(g[u])) bad_g = true;
                    if (p.mode == 0 || p.mode == 4) {
                        p.s_out[idx[u]] = g[u];
                        continue;
                    }
                    const float G = (p.mode == 1 || p.mode == 2) ? __fadd_rn(sv[u], g[u]) : g[u];
                    if (p.mode == 1) {
                        p.s_out[idx[u]] = G;
                        continue;
                    }
                    float v = p.momentum != 0.f ? vv[u] : 0.f;
                    const float nt = sgd_update(p, G, th[u], v, lr);
                    if (p.momentum != 0.f) p.vel[idx[u]] = v;
                    if (!isfinite(nt)) bad_u = true;
                    p.theta_new[idx[u]] = nt;
                    Fmt<KIND>::store(p.wc_new.hi, p.wc_new.lo, widx[u], nt);
                }
            }
        }
        if (bad_g) atomicOr(p.grad_flags, 1u << ((p.stage - 1) & 31));
        if (bad_u) atomicOr(p.upd_flags, 1u << ((p.stage - 1) & 31));
    }

    // Multi-GPU ring protocol around the hop (comm.py:37-67 made real):
    //   pre : wait until the previous rank's partial of this step is complete,
    //         until the next rank has consumed our previous partial (we are
    //         about to overwrite it), and (updater) until every reader pulled
    //         the version this update overwrites;
    //   post: the last CTA publishes ready / consumed / updated.
    // called by the 128 epilogue threads (named barrier 1)
    __device__ static void pre(const Params &p, int tid, bool external = false) {
        if (!p.sync.enabled || p.mode >= 3 || (p.sync.pre_external && !external)) return;
        if (tid == 0) {
            const uint32_t t = uint32_t(*p.sync.step), j = p.stage - 1;
            uint32_t *err = &p.sync.own->err;
            if (p.mode == 1 || p.mode == 2) spin_ge(&p.sync.prev->ready[j], t, err);
            if (p.mode == 0 || p.mode == 1) spin_ge(&p.sync.own->consumed[j], t - 1, err);
            if (p.mode == 2 && t >= 3) spin_ge(&p.sync.own->pulled[j][(t + 1) & 1], p.sync.n_readers, err);
        }
        asm volatile("bar.sync 1, 128;" ::: "memory");
    }
    __device__ static void post(const Params &p, int tid, unsigned n_ctas) {
        if (!p.sync.enabled || p.mode >= 3) return;  // single worker / gradient-only publish nothing
        __syncthreads();
        if (tid == 0) {
            const uint32_t t = uint32_t(*p.sync.step), j = p.stage - 1;
            // gpu-scope fence orders this CTA's stores before its arrival; the last
            // CTA's system-scope release is cumulative over everything it observed
            __threadfence();
            if (atomicAdd(&p.sync.cta_counter[j], 1u) == n_ctas - 1) {
                p.sync.cta_counter[j] = 0;
                __threadfence_system();
                if (p.mode == 1 || p.mode == 2) ptx::st_release_sys(&p.sync.prev->consumed[j], t);
                if (p.mode == 0 || p.mode == 1) ptx::st_release_sys(&p.sync.own->ready[j], t);
                if (p.mode == 2) {
                    p.sync.own->pulled[j][(t + 1) & 1] = 0;
                    p.sync.own->vtag[(t + 1) & 1][j] = t + 1;  // version tag of the new slot (trace mode)
                    ptx::st_release_sys(&p.sync.own->updated[j], t + 1);
                }
            }
        }
    }

    __device__ static void extra(const Params &, int, int) {}
};

// ---------------------------------------------------------------------------
// Loss + dz of the last stage (ref _kernels.pyx:64-100) for one micro-batch.
// One CTA; thread s handles sample s; the loss is reduced in ascending s.
template <int KIND>
__global__ void loss_kernel(const float *__restrict__ z, int B, int dout, int loss_kind, const int *perm,
                            const int *labels, const float *targets, CTensor dz, double *loss_out,
                            unsigned *loss_flag) {
    // shared: per-sample loss [blockDim] doubles, then dz [B][dout] floats
    extern __shared__ double sh_loss[];
    float *sdz = reinterpret_cast<float *>(sh_loss + blockDim.x);
    ptx::griddep_wait();
    ptx::griddep_launch();
    const int s = threadIdx.x;
    double l = 0.0;
    if (s < B) {
        const int row = perm[s];
        const float *zr = z + size_t(s) * dout;
        if (loss_kind == 0) {
            const float *tr = targets + size_t(row) * dout;
            for (int o = 0; o < dout; ++o) {
                const float d = __fsub_rn(zr[o], tr[o]);
                l += double(d) * double(d);
                sdz[s * dout + o] = __fdiv_rn(d, float(B));
            }
        } else {
            const int lab = labels[row];
            float mx = zr[0];
            for (int o = 1; o < dout; ++o) mx = fmaxf(mx, zr[o]);
            float se = 0.f;
            for (int o = 0; o < dout; ++o) se = __fadd_rn(se, expf(__fsub_rn(zr[o], mx)));
            for (int o = 0; o < dout; ++o) {
                const float pz = __fdiv_rn(expf(__fsub_rn(zr[o], mx)), se);
                if (o == lab) l = -log(double(pz));
                sdz[s * dout + o] = __fdiv_rn(__fsub_rn(pz, o == lab ? 1.f : 0.f), float(B));
            }
        }
        for (int o = 0; o < dout; ++o) Fmt<KIND>::store(dz.hi, dz.lo, size_t(s) * dz.ld + o, sdz[s * dout + o]);
    }
    sh_loss[s] = l;
    __syncthreads();
    if (s == 0) {
        double acc = 0.0;
        for (int k = 0; k < B; ++k) acc += sh_loss[k];
        acc = loss_kind == 0 ? acc / (2.0 * B) : acc / B;
        *loss_out = acc;
        if (!isfinite(acc)) atomicOr(loss_flag, 1u);
    }
}

// Gather micro-batch rows of the device-resident dataset into a stage-1
// input record (compute format); column din keeps the constant 1 of the
// bias-folding ones column (written once at allocation).
template <int KIND>
__global__ void gather_kernel(const float *__restrict__ data, int din, const int *perm, CTensor out) {
    ptx::griddep_wait();
    ptx::griddep_launch();
    const int s = blockIdx.x;
    const float *src = data + size_t(perm[s]) * din;
    for (int k = threadIdx.x; k < din; k += blockDim.x) Fmt<KIND>::store(out.hi, out.lo, size_t(s) * out.ld + k, src[k]);
}

// theta delivery (the step the reference plan leaves implicit):
// reader ranks copy stage j of version v from the updater's HBM over NVLink
// into their own slot v % 2 (master fp32 + packed compute copy), then count
// themselves in the updater's pulled[j][v % 2].  v = t (fresh read) or t-1.
// Versions <= 1 are the initialisation every rank already holds.
template <int KIND>
__global__ void pull_stage_kernel(const float *__restrict__ src, float *dst, int din, int dout, CTensor wc,
                                  RingFlags *updater, RingFlags *own, int stage, int fresh, const int *step,
                                  unsigned *cta_counter) {
    ptx::griddep_wait();
    ptx::griddep_launch();
    const int t = *step;
    const uint32_t v = uint32_t(fresh ? t : t - 1);
    if (v <= 1) return;
    __shared__ int go;
    if (threadIdx.x == 0) {
        spin_ge(&updater->updated[stage - 1], v, &own->err);
        go = 1;
    }
    __syncthreads();
    const int64_t n = int64_t(din + 1) * dout;  // [W; b]
    for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < n; i += int64_t(gridDim.x) * blockDim.x) {
        const float x = __ldcv(src + i);  // peer memory: bypass stale cached copies
        dst[i] = x;
        Fmt<KIND>::store(wc.hi, wc.lo, size_t(i / dout) * wc.ld + i % dout, x);
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        __threadfence_system();
        if (atomicAdd(&cta_counter[stage - 1], 1u) == gridDim.x - 1) {
            cta_counter[stage - 1] = 0;
            atomicAdd_system(&updater->pulled[stage - 1][v & 1], 1u);
        }
    }
}

// Pack a master fp32 stage ([W; b] = [din+1][dout]) into its compute copy [din+1][ld].
template <int KIND>
__global__ void pack_w_kernel(const float *__restrict__ w, int din, int dout, CTensor out) {
    const size_t n = size_t(din + 1) * dout;
    for (size_t i = blockIdx.x * size_t(blockDim.x) + threadIdx.x; i < n; i += size_t(gridDim.x) * blockDim.x) {
        const size_t k = i / dout, o = i % dout;
        Fmt<KIND>::store(out.hi, out.lo, k * out.ld + o, w[i]);
    }
}

}  // namespace cdp

namespace cdp {
// Set column `col` of a [rows][ld] compute-format record to 1 (the ones column).
template <int KIND>
__global__ void ones_column_kernel(CTensor t, int rows, int col) {
    for (int r = blockIdx.x * blockDim.x + threadIdx.x; r < rows; r += gridDim.x * blockDim.x)
        Fmt<KIND>::store(t.hi, t.lo, size_t(r) * t.ld + col, 1.f);
}
}  // namespace cdp

namespace cdp {
// DP all-reduce baseline (ref comm.py:70-90): after the collective has summed
// every rank's gradient into S, each replica applies the same update.
template <int KIND>
__global__ void update_from_sum_kernel(HopParams p) {
    ptx::griddep_wait();
    const int64_t n = int64_t(p.din + 1) * p.dout;
    const float lr = *p.lr;
    bool bad = false;
    for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < n; i += int64_t(gridDim.x) * blockDim.x) {
        const int64_t idx = p.base + i;
        float v = p.momentum != 0.f ? p.vel[idx] : 0.f;
        const float nt = sgd_update(p, p.s_in[idx], p.theta_cur[idx], v, lr);
        if (p.momentum != 0.f) p.vel[idx] = v;
        if (!isfinite(nt)) bad = true;
        p.theta_new[idx] = nt;
        Fmt<KIND>::store(p.wc_new.hi, p.wc_new.lo, size_t(i / p.dout) * p.wc_new.ld + i % p.dout, nt);
    }
    if (bad) atomicOr(p.upd_flags, 1u << ((p.stage - 1) & 31));
}
}  // namespace cdp
