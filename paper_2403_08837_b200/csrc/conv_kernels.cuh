// Convolutional-network layer kernels for the ResNet configs (BASELINE
// configs[1..2,4]).  Convolutions are tcgen05 GEMMs (gemm_pk_kernel): implicit
// (TMA-gathered NHWC boxes, MODE 1-3; stride-2 data gradients as four sub-pixel
// phases) for every conv whose input channels fill a 128-byte chunk, a plain
// GEMM for 1x1 stride-1 convs, and an explicit im2col only for the 3-channel stem.  Batch norm runs in training mode (per
// micro-batch statistics) with fixed-order reductions: the forward statistics
// come out of the conv GEMM's epilogue (per M tile), the backward ones from a
// row-blocked partial kernel; both are finalised in fp64 in a fixed order.
//
// Storage: activations in the GEMM compute format (bf16, or fp32 hi/lo for the
// 3xTF32 mode); conv outputs y and the gradients flowing between layers in
// "Y format" (bf16 in the bf16 mode, fp32 in the fp32 mode); every reduction
// and every elementwise computation in fp32 registers.  All elementwise
// kernels move 4 channels per thread.
#pragma once
#include <cstdlib>

#include "gemm_pk.cuh"
#include "mlp_kernels.cuh"

namespace cdp {

// ---------------------------------------------------------------- vector access helpers
template <int KIND>
__device__ __forceinline__ float4 ld_c4(const CTensor &t, size_t i) {
    if constexpr (KIND == 0) {
        const uint2 u = *reinterpret_cast<const uint2 *>(static_cast<const __nv_bfloat16 *>(t.hi) + i);
        const __nv_bfloat162 a = *reinterpret_cast<const __nv_bfloat162 *>(&u.x);
        const __nv_bfloat162 b = *reinterpret_cast<const __nv_bfloat162 *>(&u.y);
        const float2 fa = __bfloat1622float2(a), fb = __bfloat1622float2(b);
        return make_float4(fa.x, fa.y, fb.x, fb.y);
    } else {
        const float4 h = *reinterpret_cast<const float4 *>(static_cast<const float *>(t.hi) + i);
        const float4 l = *reinterpret_cast<const float4 *>(static_cast<const float *>(t.lo) + i);
        return make_float4(__fadd_rn(h.x, l.x), __fadd_rn(h.y, l.y), __fadd_rn(h.z, l.z), __fadd_rn(h.w, l.w));
    }
}

// Y format: bf16 (KIND 0) or fp32 (KIND 1)
template <int KIND>
__device__ __forceinline__ float4 ld_y4(const void *y, size_t i) {
    if constexpr (KIND == 0) {
        const CTensor t{const_cast<void *>(y), nullptr, 0};
        return ld_c4<0>(t, i);
    } else {
        return *reinterpret_cast<const float4 *>(static_cast<const float *>(y) + i);
    }
}
template <int KIND>
__device__ __forceinline__ void st_y4(void *y, size_t i, float4 v) {
    if constexpr (KIND == 0) {
        store_wc4<0>(CTensor{y, nullptr, 0}, i, v);
    } else {
        *reinterpret_cast<float4 *>(static_cast<float *>(y) + i) = v;
    }
}
__device__ __forceinline__ float4 relu_mask4(float4 g, float4 a) {
    return make_float4(a.x > 0.f ? g.x : 0.f, a.y > 0.f ? g.y : 0.f, a.z > 0.f ? g.z : 0.f, a.w > 0.f ? g.w : 0.f);
}
__device__ __forceinline__ float4 ld_f4(const float *p, size_t i) { return *reinterpret_cast<const float4 *>(p + i); }
__device__ __forceinline__ void st_f4(float *p, size_t i, float4 v) { *reinterpret_cast<float4 *>(p + i) = v; }

// 8-wide (16-byte bf16) vectors
struct F8 {
    float v[8];
};
__device__ __forceinline__ void bf16x8_to_f8(const uint4 u, F8 &o) {
    const uint32_t w[4] = {u.x, u.y, u.z, u.w};
#pragma unroll
    for (int k = 0; k < 4; ++k) {
        const float2 f = __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162 *>(&w[k]));
        o.v[2 * k] = f.x;
        o.v[2 * k + 1] = f.y;
    }
}
__device__ __forceinline__ uint4 f8_to_bf16x8(const F8 &a) {
    uint32_t w[4];
#pragma unroll
    for (int k = 0; k < 4; ++k) {
        __nv_bfloat162 b = __floats2bfloat162_rn(a.v[2 * k], a.v[2 * k + 1]);
        w[k] = *reinterpret_cast<uint32_t *>(&b);
    }
    return make_uint4(w[0], w[1], w[2], w[3]);
}
__device__ __forceinline__ F8 ld_f8(const float *p, size_t i) {
    F8 o;
    const float4 a = *reinterpret_cast<const float4 *>(p + i), b = *reinterpret_cast<const float4 *>(p + i + 4);
    o.v[0] = a.x, o.v[1] = a.y, o.v[2] = a.z, o.v[3] = a.w, o.v[4] = b.x, o.v[5] = b.y, o.v[6] = b.z, o.v[7] = b.w;
    return o;
}
template <int KIND>
__device__ __forceinline__ F8 ld_y8(const void *y, size_t i) {
    if constexpr (KIND == 0) {
        F8 o;
        bf16x8_to_f8(*reinterpret_cast<const uint4 *>(static_cast<const __nv_bfloat16 *>(y) + i), o);
        return o;
    } else {
        return ld_f8(static_cast<const float *>(y), i);
    }
}
template <int KIND>
__device__ __forceinline__ void st_y8(void *y, size_t i, const F8 &a) {
    if constexpr (KIND == 0) {
        *reinterpret_cast<uint4 *>(static_cast<__nv_bfloat16 *>(y) + i) = f8_to_bf16x8(a);
    } else {
        float *p = static_cast<float *>(y) + i;
        *reinterpret_cast<float4 *>(p) = make_float4(a.v[0], a.v[1], a.v[2], a.v[3]);
        *reinterpret_cast<float4 *>(p + 4) = make_float4(a.v[4], a.v[5], a.v[6], a.v[7]);
    }
}
template <int KIND>
__device__ __forceinline__ F8 ld_c8(const CTensor &t, size_t i) {
    if constexpr (KIND == 0) {
        return ld_y8<0>(t.hi, i);
    } else {
        F8 h = ld_f8(static_cast<const float *>(t.hi), i), l = ld_f8(static_cast<const float *>(t.lo), i);
#pragma unroll
        for (int k = 0; k < 8; ++k) h.v[k] = __fadd_rn(h.v[k], l.v[k]);
        return h;
    }
}
template <int KIND>
__device__ __forceinline__ void st_c8(const CTensor &t, size_t i, const F8 &a) {
    if constexpr (KIND == 0) {  // one 16-byte store (i is a multiple of 8 at every call site)
        *reinterpret_cast<uint4 *>(static_cast<__nv_bfloat16 *>(t.hi) + i) = f8_to_bf16x8(a);
    } else {
        store_wc4<KIND>(t, i, make_float4(a.v[0], a.v[1], a.v[2], a.v[3]));
        store_wc4<KIND>(t, i + 4, make_float4(a.v[4], a.v[5], a.v[6], a.v[7]));
    }
}

// ---------------------------------------------------------------------------
// Stem: gather the micro-batch's images (fp32 NHWC dataset rows, C channels)
// and im2col them in one pass: cols[p][k], k = (r*S + s)*C + c, zero padding
// and zero columns K..ld-1.  The cols matrix is the stem's activation record.
// One thread per (pixel, 8 consecutive k): 16-byte (bf16) stores.
template <int KIND, int R, int C>
static __global__ void stem_im2col_kernel(const float *__restrict__ data, const int *perm, int H, int W, int stride, int pad,
                                   int Ho, int Wo, int P, CTensor cols) {
    ptx::griddep_wait();
    ptx::griddep_launch();
    constexpr int S = R, K = R * S * C;
    const int G = cols.ld / 8;
    const int64_t n = int64_t(P) * G;
    for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < n; i += int64_t(gridDim.x) * blockDim.x) {
        const int p = int(i / G), k0 = int(i - int64_t(p) * G) * 8;
        const int wo = p % Wo, t = p / Wo, ho = t % Ho, b = t / Ho;
        const float *img = data + size_t(perm[b]) * H * W * C;
        float v[8];
#pragma unroll
        for (int j = 0; j < 8; ++j) {
            const int k = k0 + j;
            float x = 0.f;
            if (k < K) {
                const int r = k / (S * C), rem = k - r * (S * C), s = rem / C, c = rem - s * C;
                const int h = ho * stride - pad + r, w = wo * stride - pad + s;
                if (h >= 0 && h < H && w >= 0 && w < W) x = __ldg(img + (size_t(h) * W + w) * C + c);
            }
            v[j] = x;
        }
        const size_t o = size_t(p) * cols.ld + k0;
        store_wc4<KIND>(cols, o, make_float4(v[0], v[1], v[2], v[3]));
        store_wc4<KIND>(cols, o + 4, make_float4(v[4], v[5], v[6], v[7]));
    }
}

// Row-staged stem im2col: one CTA per (image, output row).  The R input rows the
// output row reads (zero-padded left / right / outside the image) are staged in
// shared memory with 16-byte loads; each thread then writes one output pixel's
// record row from them (the CTA's output rows form one contiguous [Wo][ld] block).
// (The per-element version: 0.57 ms, 0.9 TB/s, for the 514 MB ImageNet-stem record.)
// Requires (W + 2 pad) * C * R floats + ld ints of shared memory (dynamic).
template <int KIND, int R, int C>
static __global__ void __launch_bounds__(256) stem_im2col_rows_kernel(const float *__restrict__ data, const int *perm,
                                                                       int H, int W, int stride, int pad, int Ho,
                                                                       int Wo, CTensor cols) {
    ptx::griddep_wait();
    ptx::griddep_launch();
    extern __shared__ float sm_rows[];
    constexpr int S = R, K = R * S * C;
    const int Wp = W + 2 * pad;
    const int rowlen = Wp * C;
    const int ho = blockIdx.x % Ho, b = blockIdx.x / Ho;
    const float *img = data + size_t(__ldg(perm + b)) * H * W * C;
    // stage the R input rows: 16-byte loads of each row's W * C contiguous floats (one division per
    // vector, none per element: the per-element version was instruction-bound at 1.8 TB/s), zero pads
    const int WC4 = W * C / 4, padc = pad * C;
    for (int i = threadIdx.x; i < R * WC4; i += blockDim.x) {
        const int r = i / WC4, q4 = i - r * WC4;
        const int h = ho * stride - pad + r;
        float4 x = make_float4(0.f, 0.f, 0.f, 0.f);
        if (h >= 0 && h < H) x = __ldg(reinterpret_cast<const float4 *>(img + size_t(h) * W * C) + q4);
        float *d = sm_rows + r * rowlen + padc + 4 * q4;
        d[0] = x.x;
        d[1] = x.y;
        d[2] = x.z;
        d[3] = x.w;
    }
    for (int i = threadIdx.x; i < R * 2 * padc; i += blockDim.x) {
        const int r = i / (2 * padc), q = i - r * 2 * padc;
        sm_rows[r * rowlen + (q < padc ? q : padc + W * C + (q - padc))] = 0.f;
    }
    __syncthreads();
    // gather: one thread per output pixel, its K = R * S * C values in k order (per tap row r a contiguous
    // S * C run of the staged row), packed 8 at a time into 16-byte stores (no offset table: the table
    // version was shared-memory bound, 92 % MIO)
    constexpr int KP = (K + 7) / 8 * 8;
    const size_t row0 = (size_t(b) * Ho + ho) * Wo;
    for (int wo = threadIdx.x; wo < Wo; wo += blockDim.x) {
        const float *src = sm_rows + wo * stride * C;
        const size_t o = (row0 + wo) * cols.ld;
        F8 v;
#pragma unroll
        for (int k = 0; k < KP; ++k) {
            const int r = k / (S * C), rem = k - r * (S * C);
            v.v[k & 7] = k < K ? src[r * rowlen + rem] : 0.f;
            if ((k & 7) == 7) st_c8<KIND>(cols, o + k - 7, v);
        }
#pragma unroll
        for (int j = 0; j < 8; ++j) v.v[j] = 0.f;
        for (int k = KP; k < cols.ld; k += 8) st_c8<KIND>(cols, o + k, v);
    }
}

// exact-erf GELU and its derivative (torch.nn.functional.gelu default)
__device__ __forceinline__ float gelu(float x) { return 0.5f * x * (1.f + erff(x * 0.70710678118654752f)); }
__device__ __forceinline__ float gelu_grad(float x) {
    return 0.5f * (1.f + erff(x * 0.70710678118654752f)) + x * 0.39894228040143268f * __expf(-0.5f * x * x);
}
// gelu(x) and gelu'(x) from one erf (the forward stores gelu'(z) for the backward instead of z)
__device__ __forceinline__ void gelu_both(float x, float &g, float &d) {
    const float e = 0.5f * (1.f + erff(x * 0.70710678118654752f));
    g = x * e;
    d = e + x * 0.39894228040143268f * __expf(-0.5f * x * x);
}

// ---------------------------------------------------------------------------
// Epilogues of the persistent GEMM (gemm_pk_kernel / pk_reduce_kernel): run()
// gets a shared sub-tile st[nrows][ncols] (row stride lds), the row map
// rowm[r] (output row or -1) and the absolute column col0 of st's column 0.

// Conv output (Y format) or data gradient (fp32) rows, plus (stats != null) the
// tile's per-channel (sum, sum sq) over its valid rows in ascending row order
// -> stats[tile_m][N][2] (requires the whole 128-row tile in one call).
template <int KIND>
struct EpiConvOut2 {
    struct Params {
        void *out;           // Y format (bf16 / fp32): conv outputs and activation gradients
        int ld;
        float *stats;        // [N][tiles][2] (channel-major: the finalise reads it coalesced)
        int tiles;
        const void *add;     // Y-format [rows][ld] added to the output (residual gradient), or null
        CTensor add_mask;    // add masked by (add_mask > 0) when add_mask.hi
        CTensor out_mask;    // the final value masked by (out_mask > 0) when out_mask.hi (a ReLU's gradient
                             // mask applied by the producer: its consumers then read no mask)
        int out_f32;         // 1: fp32 output rows (and `add` is fp32): the ViT residual stream
        CTensor gelu_out;    // also write gelu(out) here (compute format, own ld), or null
        const void *gelu_z;  // out *= gelu'(z), z Y-format with the output's layout, or null
        const void *mul;     // out *= mul (Y format, the output's layout): a stored gelu'(z), or null
        int out_gelu_grad;   // with gelu_out: the stored output is gelu'(x) instead of x (the backward's factor)
        void *out_lo;        // KIND 1: store `out` in compute format (hi = out, lo = out_lo; a GEMM operand), or null
    };
    static constexpr int kStages = 0;
    static Params for_split(const Params &p) { return p; }
    // plain bf16 output rows (no residual / GELU / fp32 stream): the persistent kernel may store
    // the tile with TMA (gemm_pk_kernel, PkArgs::tma_out)
    static constexpr bool kTmaStore = KIND == 0;
    static bool tma_eligible(const Params &p) {
        return KIND == 0 && p.out && !p.add && !p.out_mask.hi && !p.gelu_z && !p.mul && !p.gelu_out.hi && !p.out_f32 &&
               (p.ld % 8) == 0 &&
               (reinterpret_cast<uintptr_t>(p.out) & 15) == 0;
    }
    __device__ static bool has_stats(const Params &p) { return p.stats != nullptr; }
    // Unit start (persistent kernel, one thread per tile row): pull the row's extra operands
    // (residual, mask, GELU input) into L2 while the mainloop runs.
    __device__ static void prefetch_row(const Params &p, int m, int col0, int ncols, int64_t off) {
        if (m < 0 || ((p.ld | col0 | ncols) & 7) || (off & 7)) return;
        const size_t o = size_t(off) + size_t(m) * p.ld + col0;
        const int ab = (p.out_f32 || KIND == 1) ? 4 : 2;
        if (p.add) ptx::prefetch_l2(static_cast<const char *>(p.add) + o * ab, uint32_t(ncols * ab));
        if (KIND == 0 && p.add_mask.hi) ptx::prefetch_l2(static_cast<const char *>(p.add_mask.hi) + o * 2, uint32_t(ncols * 2));
        if (KIND == 0 && p.gelu_z) ptx::prefetch_l2(static_cast<const char *>(p.gelu_z) + o * 2, uint32_t(ncols * 2));
        if (KIND == 0 && p.mul) ptx::prefetch_l2(static_cast<const char *>(p.mul) + o * 2, uint32_t(ncols * 2));
    }

    // Drain hook (per warp, lane = tile row, v = 32 consecutive columns from TMEM).
    __device__ static void drain(const Params &p, bool split, int m, int col, float (&v)[32], float *srow,
                                 float *pp) {
#pragma unroll
        for (int i = 0; i < 32; i += 4)
            *reinterpret_cast<float4 *>(srow + i) = make_float4(v[i], v[i + 1], v[i + 2], v[i + 3]);
        if (p.stats && !split) {  // squares in place, then the values again from the shared row (32 live)
#pragma unroll
            for (int i = 0; i < 32; ++i) v[i] = m >= 0 ? v[i] * v[i] : 0.f;
            pp[1] = warp_colsum32(v);
#pragma unroll
            for (int i = 0; i < 32; i += 4) {
                const float4 t = *reinterpret_cast<const float4 *>(srow + i);
                v[i] = m >= 0 ? t.x : 0.f;
                v[i + 1] = m >= 0 ? t.y : 0.f;
                v[i + 2] = m >= 0 ? t.z : 0.f;
                v[i + 3] = m >= 0 ? t.w : 0.f;
            }
            pp[0] = warp_colsum32(v);
        }
    }
    // Stores (8 columns per element: 16-byte bf16 / 2 x 16-byte fp32 stores).
    // FIXC: ncols known at compile time (the persistent kernel's full passes), 0 = runtime.
    // TAIL: aligned rows keep the 8-column vectors up to the last full vector and only the columns
    // past it (a 197-token tile) take the scalar loop; otherwise a ragged ncols makes the whole tile
    // scalar (fewer live registers: the split-K reduce kernel keeps its occupancy).
    template <int NTH, int FIXC = 0, bool TAIL = false>
    __device__ static void run(const Params &p, const float *st, int lds, const int *rowm, int nrows, int col0,
                               int ncols, int tm, int N, int tid, int64_t off) {
        if (FIXC) ncols = FIXC;
        const bool rows_aligned = !(((p.ld | col0) & 7) || (off & 7));
        int nv = ncols;  // columns of the 8-wide vector path
        if (!rows_aligned || (ncols & 7)) {
            nv = (TAIL && rows_aligned) ? (ncols & ~7) : 0;
            const int nt = ncols - nv;
            for (int e = tid; e < nrows * nt; e += NTH) {
                const int r = e / nt, c = nv + (e - r * nt);
                const int m = rowm[r];
                if (m < 0) continue;
                float x = st[r * lds + c];
                const size_t o = size_t(off) + size_t(m) * p.ld + col0 + c;
                if (p.add) {
                    float a = p.out_f32 ? static_cast<const float *>(p.add)[o] : Fmt<0>::load(p.add, nullptr, o);
                    if (KIND == 1 && !p.out_f32) a = static_cast<const float *>(p.add)[o];
                    if (p.add_mask.hi && !(Fmt<KIND>::load(p.add_mask.hi, p.add_mask.lo, o) > 0.f)) a = 0.f;
                    x += a;
                }
                if (p.out_mask.hi && !(Fmt<KIND>::load(p.out_mask.hi, p.out_mask.lo, o) > 0.f)) x = 0.f;
                if (p.gelu_z) x *= gelu_grad(KIND == 0 ? Fmt<0>::load(p.gelu_z, nullptr, o)
                                                       : static_cast<const float *>(p.gelu_z)[o]);
                if (p.mul) x *= KIND == 0 ? Fmt<0>::load(p.mul, nullptr, o) : static_cast<const float *>(p.mul)[o];
                if (p.gelu_out.hi) {
                    float gl, gd;
                    gelu_both(x, gl, gd);
                    Fmt<KIND>::store(p.gelu_out.hi, p.gelu_out.lo, size_t(m) * p.gelu_out.ld + col0 + c, gl);
                    if (p.out_gelu_grad) x = gd;
                }
                if (KIND == 1 && p.out_lo && !p.out_f32)
                    Fmt<1>::store(p.out, p.out_lo, o, x);
                else if (p.out_f32 || KIND == 1)
                    static_cast<float *>(p.out)[o] = x;
                else
                    Fmt<0>::store(p.out, nullptr, o, x);
            }
            if (!TAIL || nv == 0) return;
        }
        const int C8 = FIXC ? FIXC / 8 : nv / 8;
        const int total = nrows * C8;
        constexpr int U = 2;
        for (int e0 = tid; e0 < total; e0 += NTH * U) {
            float4 v[U][2], a[U][2], mk[U][2];
            size_t o[U];
            int gm[U], gc[U];
            bool ok[U];
#pragma unroll
            for (int u = 0; u < U; ++u) {
                const int e = e0 + u * NTH;
                const int r = e / C8, c = (e - r * C8) * 8;
                ok[u] = e < total && rowm[r] >= 0;
                if (!ok[u]) continue;
                v[u][0] = *reinterpret_cast<const float4 *>(st + r * lds + c);
                v[u][1] = *reinterpret_cast<const float4 *>(st + r * lds + c + 4);
                o[u] = size_t(off) + size_t(rowm[r]) * p.ld + col0 + c;
                gm[u] = rowm[r];
                gc[u] = col0 + c;
                if (p.add) {
                    if (p.out_f32) {
                        a[u][0] = ld_f4(static_cast<const float *>(p.add), o[u]);
                        a[u][1] = ld_f4(static_cast<const float *>(p.add), o[u] + 4);
                    } else {
                        a[u][0] = ld_y4<KIND>(p.add, o[u]);
                        a[u][1] = ld_y4<KIND>(p.add, o[u] + 4);
                    }
                }
                if (p.add_mask.hi || p.out_mask.hi) {  // exclusive: one mask register set
                    const CTensor &mt = p.add_mask.hi ? p.add_mask : p.out_mask;
                    mk[u][0] = ld_c4<KIND>(mt, o[u]);
                    mk[u][1] = ld_c4<KIND>(mt, o[u] + 4);
                }
            }
#pragma unroll
            for (int u = 0; u < U; ++u) {
                if (!ok[u]) continue;
#pragma unroll
                for (int k = 0; k < 2; ++k) {
                    if (p.add) {
                        const float4 b = p.add_mask.hi ? relu_mask4(a[u][k], mk[u][k]) : a[u][k];
                        v[u][k].x += b.x;
                        v[u][k].y += b.y;
                        v[u][k].z += b.z;
                        v[u][k].w += b.w;
                    }
                    if (p.out_mask.hi) v[u][k] = relu_mask4(v[u][k], mk[u][k]);
                }
                if (p.gelu_z || p.mul) {  // (exclusive) gelu'(z) from z, or a stored factor
                    const F8 zz = ld_y8<KIND>(p.gelu_z ? p.gelu_z : p.mul, o[u]);
                    float w8[8] = {v[u][0].x, v[u][0].y, v[u][0].z, v[u][0].w,
                                   v[u][1].x, v[u][1].y, v[u][1].z, v[u][1].w};
#pragma unroll
                    for (int i = 0; i < 8; ++i) w8[i] *= p.gelu_z ? gelu_grad(zz.v[i]) : zz.v[i];
                    v[u][0] = make_float4(w8[0], w8[1], w8[2], w8[3]);
                    v[u][1] = make_float4(w8[4], w8[5], w8[6], w8[7]);
                }
                if (p.gelu_out.hi) {
                    const size_t og = size_t(gm[u]) * p.gelu_out.ld + gc[u];
                    float w8[8] = {v[u][0].x, v[u][0].y, v[u][0].z, v[u][0].w,
                                   v[u][1].x, v[u][1].y, v[u][1].z, v[u][1].w};
                    float g8[8];
#pragma unroll
                    for (int i = 0; i < 8; ++i) gelu_both(w8[i], g8[i], w8[i]);  // w8: gelu'(x) from here on
                    store_wc4<KIND>(p.gelu_out, og, make_float4(g8[0], g8[1], g8[2], g8[3]));
                    store_wc4<KIND>(p.gelu_out, og + 4, make_float4(g8[4], g8[5], g8[6], g8[7]));
                    if (p.out_gelu_grad) {
                        v[u][0] = make_float4(w8[0], w8[1], w8[2], w8[3]);
                        v[u][1] = make_float4(w8[4], w8[5], w8[6], w8[7]);
                    }
                }
                if (p.out_f32) {
                    st_f4(static_cast<float *>(p.out), o[u], v[u][0]);
                    st_f4(static_cast<float *>(p.out), o[u] + 4, v[u][1]);
                } else if (KIND == 0) {
                    __nv_bfloat162 b0 = __floats2bfloat162_rn(v[u][0].x, v[u][0].y);
                    __nv_bfloat162 b1 = __floats2bfloat162_rn(v[u][0].z, v[u][0].w);
                    __nv_bfloat162 b2 = __floats2bfloat162_rn(v[u][1].x, v[u][1].y);
                    __nv_bfloat162 b3 = __floats2bfloat162_rn(v[u][1].z, v[u][1].w);
                    uint4 w;
                    w.x = *reinterpret_cast<uint32_t *>(&b0);
                    w.y = *reinterpret_cast<uint32_t *>(&b1);
                    w.z = *reinterpret_cast<uint32_t *>(&b2);
                    w.w = *reinterpret_cast<uint32_t *>(&b3);
                    *reinterpret_cast<uint4 *>(static_cast<__nv_bfloat16 *>(p.out) + o[u]) = w;
                } else if (p.out_lo) {  // KIND 1 compute format
                    store_wc4<KIND>(CTensor{p.out, p.out_lo, 0}, o[u], v[u][0]);
                    store_wc4<KIND>(CTensor{p.out, p.out_lo, 0}, o[u] + 4, v[u][1]);
                } else {
                    st_y4<KIND>(p.out, o[u], v[u][0]);
                    st_y4<KIND>(p.out, o[u] + 4, v[u][1]);
                }
            }
        }
    }
    // Persistent kernel: the CTA's running per-column (sum, sum sq) over its units (in
    // its fixed unit order) lives in stats[c][blockIdx.x][2]; col_stats_init zeroes the
    // CTA's slice, col_stats adds the 4 TMEM-quarter partials of a unit (fixed order).
    // Column a is always handled by epilogue thread a % pcols (program order, no race).
    template <int NTH>
    __device__ static void col_stats_init(const Params &p, int N, int pcols, int tid) {
        if (tid >= pcols) return;
        if (p.stats)
            for (int a = tid; a < N; a += pcols)
                *reinterpret_cast<float2 *>(p.stats + (size_t(a) * gridDim.x + blockIdx.x) * 2) = make_float2(0.f, 0.f);
    }
    // The running value of the thread's column, loaded before the unit's accumulator is
    // ready (hides the load latency; the same thread stored it at its previous unit).
    // (an 8-byte cp.async into the thread's own shared slot: a register load here was spilled and its
    // wait stalled the epilogue at every unit start)
    __device__ static void col_stats_pre(const Params &p, int col0, int ncols, int tid, float *slot) {
        if (!p.stats || tid >= ncols) return;
        ptx::cp_async8(slot + 2 * tid, p.stats + (size_t(col0 + tid) * gridDim.x + blockIdx.x) * 2);
        ptx::cp_async_commit();
    }
    // TMA-store epilogue: the unit's column sums were reduced from the bf16 staging tile into
    // part[8 warps][pcols][2] (gemm_pk_kernel, pk_tile_stats); thread `tid` adds its column's eight
    // warp partials in warp order to the running value.
    __device__ static void col_stats8(const Params &p, const float *part, int pcols, int col0, int ncols, int tid,
                                      const float *slot) {
        if (p.stats && tid < ncols) {
            ptx::cp_async_wait_all();
            const float2 cur = *reinterpret_cast<const float2 *>(slot + 2 * tid);
            float s = 0.f, q = 0.f;
#pragma unroll
            for (int w = 0; w < 8; ++w) {
                const float2 t = *reinterpret_cast<const float2 *>(part + (w * pcols + tid) * 2);
                s += t.x;
                q += t.y;
            }
            *reinterpret_cast<float2 *>(p.stats + (size_t(col0 + tid) * gridDim.x + blockIdx.x) * 2) =
                make_float2(cur.x + s, cur.y + q);
        }
    }
    // Grouped TMA-store epilogue (PkArgs::grouped): each 128-thread group of epilogue warps keeps its own
    // running statistics in slot sl of nsl = 2 * gridDim.x per column; thread gt owns columns gt + 128 k.
    __device__ static void gstats_init(const Params &p, int N, int gt, int nsl, int sl) {
        if (p.stats)
            for (int a = gt; a < N; a += 128)
                *reinterpret_cast<float2 *>(p.stats + (size_t(a) * nsl + sl) * 2) = make_float2(0.f, 0.f);
    }
    __device__ static void gstats_pre(const Params &p, int col0, int ncols, int gt, float *slot, int nsl, int sl) {
        if (!p.stats || gt >= ncols) return;
        ptx::cp_async8(slot + 2 * gt, p.stats + (size_t(col0 + gt) * nsl + sl) * 2);
        ptx::cp_async_commit();
    }
    // the group's four warp partials part[4][pcols][2] in warp order, added to the running value
    __device__ static void gstats_add(const Params &p, const float *part, int pcols, int col0, int ncols, int gt,
                                      const float *slot, int nsl, int sl) {
        if (p.stats && gt < ncols) {
            ptx::cp_async_wait_all();
            const float2 cur = *reinterpret_cast<const float2 *>(slot + 2 * gt);
            float s = 0.f, q = 0.f;
#pragma unroll
            for (int w = 0; w < 4; ++w) {
                const float2 t = *reinterpret_cast<const float2 *>(part + (w * pcols + gt) * 2);
                s += t.x;
                q += t.y;
            }
            *reinterpret_cast<float2 *>(p.stats + (size_t(col0 + gt) * nsl + sl) * 2) = make_float2(cur.x + s, cur.y + q);
        }
    }
    // tensor-core statistics: the thread's column sum / sum of squares of the unit, added to the running value
    __device__ static void col_stats_value(const Params &p, int col0, int ncols, int tid, float s, float q,
                                           const float *slot) {
        if (p.stats && tid < ncols) {
            ptx::cp_async_wait_all();
            const float2 cur = *reinterpret_cast<const float2 *>(slot + 2 * tid);
            *reinterpret_cast<float2 *>(p.stats + (size_t(col0 + tid) * gridDim.x + blockIdx.x) * 2) =
                make_float2(cur.x + s, cur.y + q);
        }
    }
    template <int NTH>  // one column per thread (ncols <= NTH)
    __device__ static void col_stats(const Params &p, const float *part, int pcols, int col0, int ncols, int tm,
                                     int tid, const float *slot) {
        if (p.stats && tid < ncols) {
            ptx::cp_async_wait_all();
            const float2 cur = *reinterpret_cast<const float2 *>(slot + 2 * tid);
            float s = 0.f, q = 0.f;
#pragma unroll
            for (int k = 0; k < 4; ++k) {
                s += part[(k * pcols + tid) * 3];
                q += part[(k * pcols + tid) * 3 + 1];
            }
            *reinterpret_cast<float2 *>(p.stats + (size_t(col0 + tid) * gridDim.x + blockIdx.x) * 2) =
                make_float2(cur.x + s, cur.y + q);
        }
    }
    // Split-K reduce kernel: the whole 128-row tile is in `st` (rows in order).  Column
    // statistics: NTH/ncols row groups per column, combined in group order (fixed).
    template <int NTH>
    __device__ static void run_with_stats(const Params &p, const float *st, int lds, const int *rowm, int nrows,
                                          int col0, int ncols, int tm, int N, int tid, int64_t off) {
        run<NTH>(p, st, lds, rowm, nrows, col0, ncols, tm, N, tid, off);
        if (p.stats) {
            __shared__ float red[2][NTH];
            const int groups = NTH / ncols;
            const int c = tid % ncols, grp = tid / ncols;
            float s = 0.f, q = 0.f;
            if (grp < groups)
                for (int r = grp; r < nrows; r += groups) {
                    if (rowm[r] < 0) continue;
                    const float v = st[r * lds + c];
                    s += v;
                    q = fmaf(v, v, q);
                }
            red[0][tid] = s;
            red[1][tid] = q;
            __syncthreads();
            if (tid < ncols) {
                float a = 0.f, b = 0.f;
                for (int g = 0; g < groups; ++g) {
                    a += red[0][g * ncols + tid];
                    b += red[1][g * ncols + tid];
                }
                float *o = p.stats + (size_t(col0 + tid) * p.tiles + tm) * 2;
                o[0] = a;
                o[1] = b;
            }
        }
    }
    template <int NTH>
    __device__ static void done(const Params &, int, unsigned) {}
};

// Direct epilogue of the bf16 residual-gradient add (the ResNet block-input data gradient,
// out may alias add): EpiConvOut2's output rows with `add` (and `add_mask`), no statistics,
// no split-K.  gemm_pk_kernel instantiates ONLY the direct path for it (kDirect): each drained
// accumulator row (lane = row, 16 columns per step) is combined with its own row's residual /
// mask and stored from registers — no shared tile, no second pass over the tile.  (In the
// general epilogue the shared-tile round trip plus the dependent residual loads made the 1x1
// data gradients of ResNet-50 run at 1.9 TB/s; a direct branch inside the general kernel
// spills: its own instantiation keeps the register budget.)
template <int KIND>
struct EpiConvAdd : EpiConvOut2<KIND> {
    using Params = typename EpiConvOut2<KIND>::Params;
    static constexpr bool kDirect = true;
    static constexpr bool kTmaStore = false;
    static constexpr bool kNoSplit = true;
    static bool eligible(const Params &p, int N, int BN) {
        return KIND == 0 && (p.add != nullptr) != (p.mul != nullptr) && !p.stats && !p.out_f32 && !p.gelu_z &&
               !p.gelu_out.hi && !(p.mul && (p.add_mask.hi || p.out_mask.hi)) && (p.ld % 8) == 0 && N % BN == 0 &&
               (reinterpret_cast<uintptr_t>(p.out) & 15) == 0;
    }
    // combine mode of the row operands: 0 add, 1 add masked residual, 2 add then mask, 3 multiply (p.mul)
    __host__ __device__ static int mode(const Params &p) {
        return p.mul ? 3 : p.add_mask.hi ? 1 : p.out_mask.hi ? 2 : 0;
    }
    // Direct epilogue (bf16 residual-gradient add: the ResNet block-input data gradient, out may
    // alias add): the drained accumulator row (lane = row, 32 columns) is combined with its own
    // row's residual (and mask) and stored from registers — no shared tile, no second pass.  The
    // row's 64-byte residual / mask segments are loaded before the TMEM read (eight 16-byte loads
    // in flight per thread): with K = 64..512 this epilogue has almost no MMA work to hide behind,
    // and its L2 round trips were the kernel (1.9 TB/s in the shared-tile path).
    // 64 columns (one thread's half of an epilogue pass) per load: eight 16-byte vectors of residual
    // and eight of mask in flight per thread, issued BEFORE the accumulator is ready (they depend on
    // the row only) — the stall profile of the 16-column version was the first use of these loads
    struct DirectPre {
        uint4 a[8], m[8];
    };
    template <int NC>  // NC = 32 or 64 columns
    __device__ static void direct_load(const Params &p, int m, int col, int64_t off, DirectPre &d) {
        static_assert(NC == 32 || NC == 64, "direct epilogue loads 32 or 64 columns");
        if (m < 0) return;
        const size_t o = size_t(off) + size_t(m) * p.ld + col;
        const uint4 *pa = reinterpret_cast<const uint4 *>(static_cast<const __nv_bfloat16 *>(p.add ? p.add : p.mul) + o);
#pragma unroll
        for (int i = 0; i < NC / 8; ++i) d.a[i] = pa[i];
        if (p.add_mask.hi || p.out_mask.hi) {
            const void *mp = p.add_mask.hi ? p.add_mask.hi : p.out_mask.hi;
            const uint4 *pm = reinterpret_cast<const uint4 *>(static_cast<const __nv_bfloat16 *>(mp) + o);
#pragma unroll
            for (int i = 0; i < NC / 8; ++i) d.m[i] = pm[i];
        }
    }
    // accumulator + residual for vector u of the loaded row; mask 0: none, 1: masks the residual,
    // 2: masks the sum (the ReLU gradient mask of the output)
    __device__ static F8 combine(const DirectPre &d, int u, int mask, const float *v) {
        F8 a, x;
        bf16x8_to_f8(d.a[u], a);
        if (mask == 3) {  // the row operand is a factor (a stored gelu'(z))
#pragma unroll
            for (int k = 0; k < 8; ++k) x.v[k] = v[k] * a.v[k];
            return x;
        }
        if (mask) {
            F8 mk;
            bf16x8_to_f8(d.m[u], mk);
            if (mask == 1) {
#pragma unroll
                for (int k = 0; k < 8; ++k) x.v[k] = v[k] + (mk.v[k] > 0.f ? a.v[k] : 0.f);
            } else {
#pragma unroll
                for (int k = 0; k < 8; ++k) x.v[k] = mk.v[k] > 0.f ? v[k] + a.v[k] : 0.f;
            }
        } else {
#pragma unroll
            for (int k = 0; k < 8; ++k) x.v[k] = v[k] + a.v[k];
        }
        return x;
    }
    // columns [col + 16 q, col + 16 q + 16) of the 64 loaded ones, from v[16] (TMEM)
    __device__ static void direct_store(const Params &p, int m, int col, int q, int64_t off, const DirectPre &d,
                                        const float (&v)[16]) {
        if (m < 0) return;
        const size_t o = size_t(off) + size_t(m) * p.ld + col + 16 * q;
        uint4 *po = reinterpret_cast<uint4 *>(static_cast<__nv_bfloat16 *>(p.out) + o);
#pragma unroll
        for (int i = 0; i < 2; ++i) {
            po[i] = f8_to_bf16x8(combine(d, 2 * q + i, mode(p), v + 8 * i));
        }
    }
};

// EpiConvAdd with the residual gradient / mask rows staged into shared memory by TMA (warp 3 of
// gemm_pk_kernel issues one 64-column x 128-row box of each per chunk, kEbufSlots chunks ahead):
// the epilogue threads no longer wait on their own global loads (the ncu profile of the register
// version: 40 % of warp samples in long-scoreboard stalls on those loads, 3.0 TB/s).  BN >= 128.
template <int KIND>
struct EpiConvAddT : EpiConvAdd<KIND> {
    using Params = typename EpiConvOut2<KIND>::Params;
    using DirectPre = typename EpiConvAdd<KIND>::DirectPre;
    static constexpr bool kTmaAdd = true;
    static constexpr int kEbufSlots = 3;
    static constexpr int kStages = 2;  // mainloop ring depth (the operand ring takes the rest)
    // the thread's row (64 columns) of a 128-byte-swizzled slot: residual at +0, mask at +16 KB
    __device__ static void smem_load(const uint8_t *slot, int row, bool mask, DirectPre &d) {
        const uint8_t *ra = slot + row * 128;
#pragma unroll
        for (int i = 0; i < 8; ++i) d.a[i] = *reinterpret_cast<const uint4 *>(ra + ((i ^ (row & 7)) << 4));
        if (mask) {
            const uint8_t *rm = ra + 16384;
#pragma unroll
            for (int i = 0; i < 8; ++i) d.m[i] = *reinterpret_cast<const uint4 *>(rm + ((i ^ (row & 7)) << 4));
        }
    }
    // columns [16 q, 16 q + 16) of the chunk: accumulator + (masked) residual, written as bf16 over the
    // residual in the slot (same swizzle: the slot's first 16 KB is then the output box of a TMA store)
    __device__ static void smem_store(uint8_t *slot, int row, int q, int mask, const DirectPre &d,
                                      const float (&v)[16]) {
        uint8_t *ra = slot + row * 128;
#pragma unroll
        for (int i = 0; i < 2; ++i)
            *reinterpret_cast<uint4 *>(ra + (((2 * q + i) ^ (row & 7)) << 4)) =
                f8_to_bf16x8(EpiConvAdd<KIND>::combine(d, 2 * q + i, mask, v + 8 * i));
    }
};

// Weight gradient fused with the CDP hop / SGD update (same modes, arithmetic
// and ring protocol as EpiWgrad; the pre-hop waits run in hop_wait_kernel).
template <int KIND>
struct EpiHop2 {
    using Params = HopParams;
    static constexpr int kStages = 0;
    static Params for_split(const Params &p) { return p; }
    static constexpr bool kTmaStore = false;
    // Unit start: pull the row's optimizer state (partial sum, theta, velocity) into L2.
    __device__ static void prefetch_row(const Params &p, int m, int col0, int ncols, int64_t) {
        if (m < 0 || (p.dout % 4) || (p.base % 4) || (col0 % 4) || (ncols % 4)) return;
        const int64_t idx = p.base + int64_t(m) * p.dout + col0;
        const uint32_t bytes = uint32_t(ncols) * 4;
        if (p.mode == 1 || p.mode == 2) ptx::prefetch_l2(p.s_in + idx, bytes);
        if (p.mode == 2 || p.mode == 3) {
            ptx::prefetch_l2(p.theta_cur + idx, bytes);
            if (p.momentum != 0.f) ptx::prefetch_l2(p.vel + idx, bytes);
        }
    }
    __device__ static void drain(const Params &, bool, int, int, float (&v)[32], float *srow, float *) {
#pragma unroll
        for (int i = 0; i < 32; i += 4)
            *reinterpret_cast<float4 *>(srow + i) = make_float4(v[i], v[i + 1], v[i + 2], v[i + 3]);
    }
    __device__ static void col_stats_pre(const Params &, int, int, int, float *) {}
    template <int NTH>
    __device__ static void col_stats(const Params &, const float *, int, int, int, int, int, const float *) {}
    template <int NTH>
    __device__ static void col_stats_init(const Params &, int, int, int) {}
    template <int NTH>
    __device__ static void run_with_stats(const Params &p, const float *st, int lds, const int *rowm, int nrows,
                                          int col0, int ncols, int tm, int N, int tid, int64_t off) {
        run<NTH>(p, st, lds, rowm, nrows, col0, ncols, tm, N, tid, off);
    }
    template <int NTH, int FIXC = 0, bool TAIL = false>
    __device__ static void run(const Params &p, const float *st, int lds, const int *rowm, int nrows, int col0,
                               int ncols, int, int, int tid, int64_t) {  // FIXC / TAIL unused (register pressure)
        bool bad_g = false, bad_u = false;
        const float lr = *p.lr;
        if ((p.dout % 4) == 0 && (p.base % 4) == 0 && (ncols % 4) == 0) {
            const int C4 = ncols / 4;
            const int total = nrows * C4;
            constexpr int U = 2;
            for (int e0 = tid; e0 < total; e0 += NTH * U) {
                float4 g[U], s[U], th[U], vv[U];
                int64_t idx[U];
                size_t widx[U];
                bool ok[U];
#pragma unroll
                for (int u = 0; u < U; ++u) {
                    const int e = e0 + u * NTH;
                    const int r = e / C4, c = (e - r * C4) * 4;
                    ok[u] = e < total && rowm[r] >= 0;
                    if (!ok[u]) continue;
                    const int m = rowm[r], n = col0 + c;
                    idx[u] = p.base + int64_t(m) * p.dout + n;
                    widx[u] = size_t(m) * p.wc_new.ld + n;
                    g[u] = *reinterpret_cast<const float4 *>(st + r * lds + c);
                    if (p.mode == 1 || p.mode == 2) s[u] = __ldcg(reinterpret_cast<const float4 *>(p.s_in + idx[u]));
                    if (p.mode == 2 || p.mode == 3) {
                        th[u] = *reinterpret_cast<const float4 *>(p.theta_cur + idx[u]);
                        if (p.momentum != 0.f) vv[u] = *reinterpret_cast<const float4 *>(p.vel + idx[u]);
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
            for (int e = tid; e < nrows * ncols; e += NTH) {
                const int r = e / ncols, c = e - r * ncols;
                if (rowm[r] < 0) continue;
                hop_elem<KIND>(p, p.base + int64_t(rowm[r]) * p.dout + col0 + c, st[r * lds + c],
                               size_t(rowm[r]) * p.wc_new.ld + col0 + c, true, bad_g, bad_u);
            }
        }
        if (bad_g) atomicOr(p.grad_flags, 1u << ((p.stage - 1) & 31));
        if (bad_u) atomicOr(p.upd_flags, 1u << ((p.stage - 1) & 31));
    }
    // ring protocol: the last of `arrivals` epilogue invocations of this tensor publishes
    template <int NTH>
    __device__ static void done(const Params &p, int tid, unsigned arrivals) {
        if (!p.sync.enabled || p.mode >= 3) return;
        pk_bar(2, NTH);
        if (tid == 0) {
            const uint32_t t = uint32_t(*p.sync.step), j = p.stage - 1;
            __threadfence();
            if (atomicAdd(&p.sync.cta_counter[j], 1u) == arrivals - 1) {
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
};

// ---------------------------------------------------------------------------
// Batch norm (training mode).
// Forward finalise: per channel, the per-tile (sum, sum sq) [C][tiles][2] (fp64)
// -> mean, rstd (biased variance, eps).  One warp per channel, lanes take tiles
// lane, lane+32, ... then a fixed xor-tree: deterministic.
static __global__ void bn_finalize_fwd_kernel(const float *__restrict__ stats, int tiles, int C, int64_t P, float eps,
                                       float *mean, float *rstd) {
    ptx::griddep_wait();
    ptx::griddep_launch();
    const int c = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const int lane = threadIdx.x & 31;
    if (c >= C) return;
    double s0 = 0.0, s1 = 0.0;
    const float2 *sc = reinterpret_cast<const float2 *>(stats) + size_t(c) * tiles;  // [C][tiles] (sum, sum sq)
    for (int t = lane; t < tiles; t += 32) {
        const float2 v = sc[t];
        s0 += double(v.x);
        s1 += double(v.y);
    }
#pragma unroll
    for (int o = 16; o; o >>= 1) {
        s0 += __shfl_xor_sync(0xffffffffu, s0, o);
        s1 += __shfl_xor_sync(0xffffffffu, s1, o);
    }
    if (lane == 0) {
        const double mu = s0 / double(P);
        const double var = fmax(s1 / double(P) - mu * mu, 0.0);
        mean[c] = float(mu);
        rstd[c] = float(1.0 / sqrt(var + double(eps)));
    }
}

// y = relu?( gamma * (x - mean) * rstd + beta  [+ residual] ) -> compute format.
// residual: a compute-format tensor (identity shortcut) or a second BN-normalised
// conv output (projection shortcut).
struct BnResidual {
    CTensor act;      // identity shortcut (act.hi != null)
    const void *y;    // projection: conv output (Y format), its stats and affine
    const float *mean, *rstd, *gamma, *beta;
};

// Per-channel affine of the normalisation for 8 channels.  bf16 mode: y_hat * gamma + beta
// = x * a + b with a = gamma * rstd, b = beta - mean * a (one FMA per element, 16 registers;
// the bf16 input has far less precision than the fp32 rounding of b).  fp32 (3xTF32 parity)
// mode keeps gamma * ((x - mean) * rstd) + beta exactly as the restatement computes it.
template <int KIND>
struct BnAff {
    F8 a, b, g, e;  // KIND 0: a, b; KIND 1: a = mean, b = rstd, g = gamma, e = beta
    __device__ __forceinline__ void load(const float *mean, const float *rstd, const float *gamma, const float *beta,
                                         int c) {
        if constexpr (KIND == 0) {
            const F8 mu = ld_f8(mean, c), rs = ld_f8(rstd, c), ga = ld_f8(gamma, c), be = ld_f8(beta, c);
#pragma unroll
            for (int k = 0; k < 8; ++k) {
                a.v[k] = ga.v[k] * rs.v[k];
                b.v[k] = fmaf(-mu.v[k], a.v[k], be.v[k]);
            }
        } else {
            a = ld_f8(mean, c);
            b = ld_f8(rstd, c);
            g = ld_f8(gamma, c);
            e = ld_f8(beta, c);
        }
    }
    __device__ __forceinline__ float operator()(float x, int k) const {
        if constexpr (KIND == 0)
            return fmaf(x, a.v[k], b.v[k]);
        else
            return g.v[k] * ((x - a.v[k]) * b.v[k]) + e.v[k];
    }
};

// RES: 0 none, 1 identity shortcut (compute-format act), 2 projection shortcut (a second
// BN-normalised conv output).  One thread keeps its 8 channels (their coefficients in
// registers) for the whole grid-stride loop when the stride is a multiple of C/8 (always,
// for 256-thread blocks and C <= 2048); two vectors per iteration in flight.  The
// residual kinds are separate instantiations so the plain one keeps its registers low
// (occupancy: the generic version held 96 registers, 2 blocks / SM, 3 TB/s).
template <int KIND, int RES>
__device__ __forceinline__ void bn_apply_vec(const void *__restrict__ y, size_t o, const BnAff<KIND> &f,
                                             const BnResidual &res, const BnAff<KIND> &f2, int relu, CTensor out) {
    F8 v = ld_y8<KIND>(y, o);
#pragma unroll
    for (int k = 0; k < 8; ++k) v.v[k] = f(v.v[k], k);
    if constexpr (RES == 1) {
        const F8 r = ld_c8<KIND>(res.act, o);
#pragma unroll
        for (int k = 0; k < 8; ++k) v.v[k] += r.v[k];
    } else if constexpr (RES == 2) {
        const F8 r = ld_y8<KIND>(res.y, o);
#pragma unroll
        for (int k = 0; k < 8; ++k) v.v[k] += f2(r.v[k], k);
    }
    if (relu) {
#pragma unroll
        for (int k = 0; k < 8; ++k) v.v[k] = fmaxf(v.v[k], 0.f);
    }
    st_c8<KIND>(out, o, v);
}

template <int KIND, int RES>
static __global__ void __launch_bounds__(256) bn_apply_kernel(const void *__restrict__ y, int64_t P, int C,
                                                              const float *mean, const float *rstd,
                                                              const float *gamma, const float *beta, BnResidual res,
                                                              int relu, CTensor out) {
    ptx::griddep_wait();
    ptx::griddep_launch();
    const int C8 = C / 8;
    const int64_t n = P * C8;
    const int64_t stride = int64_t(gridDim.x) * blockDim.x;
    int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x;
    const bool fixed = stride % C8 == 0;
    BnAff<KIND> f, f2;
    f.load(mean, rstd, gamma, beta, int(i % C8) * 8);
    if constexpr (RES == 2) f2.load(res.mean, res.rstd, res.gamma, res.beta, int(i % C8) * 8);
    if (fixed) {
        if constexpr (KIND == 0) {
            // U vectors' loads issued before any store (the compiler cannot move a load above a store to
            // `out`, which it must assume may alias: one vector in flight per thread otherwise)
            constexpr int U = RES == 0 ? 4 : 2;
            const uint4 *yv = static_cast<const uint4 *>(y);
            const uint4 *rv = RES == 1 ? static_cast<const uint4 *>(res.act.hi)
                                       : RES == 2 ? static_cast<const uint4 *>(res.y) : nullptr;
            for (; i < n; i += stride * U) {
                uint4 a[U], r[U];
#pragma unroll
                for (int u = 0; u < U; ++u) {
                    const int64_t j = i + u * stride;
                    if (j < n) {
                        a[u] = yv[j];
                        if constexpr (RES != 0) r[u] = rv[j];
                    }
                }
#pragma unroll
                for (int u = 0; u < U; ++u) {
                    const int64_t j = i + u * stride;
                    if (j >= n) break;
                    F8 v;
                    bf16x8_to_f8(a[u], v);
#pragma unroll
                    for (int k = 0; k < 8; ++k) v.v[k] = f(v.v[k], k);
                    if constexpr (RES != 0) {
                        F8 q;
                        bf16x8_to_f8(r[u], q);
#pragma unroll
                        for (int k = 0; k < 8; ++k) v.v[k] += RES == 1 ? q.v[k] : f2(q.v[k], k);
                    }
                    if (relu) {
#pragma unroll
                        for (int k = 0; k < 8; ++k) v.v[k] = fmaxf(v.v[k], 0.f);
                    }
                    static_cast<uint4 *>(out.hi)[j] = f8_to_bf16x8(v);
                }
            }
            return;
        }
#pragma unroll 2
        for (; i < n; i += stride) bn_apply_vec<KIND, RES>(y, size_t(i) * 8, f, res, f2, relu, out);
        return;
    }
    for (; i < n; i += stride) {
        const int c = int(i % C8) * 8;
        f.load(mean, rstd, gamma, beta, c);
        if constexpr (RES == 2) f2.load(res.mean, res.rstd, res.gamma, res.beta, c);
        bn_apply_vec<KIND, RES>(y, size_t(i) * 8, f, res, f2, relu, out);
    }
}

// Backward statistics: per row block (ROWS rows), per channel,
// (sum g', sum g' * xhat) with g' = g masked by (act > 0) when mask != null.
// TPR threads per row (4 channels each), 256/TPR row phases; the phases are
// combined in fixed order in fp64 -> partial[C][blocks][2].  A second conv
// output (projection shortcut: same g', own y / stats) gives partial2.
constexpr int kBnRows = 256;     // largest row block
constexpr int kBnRowsMin = 64;   // smallest row block (the partial buffers are sized for it)
// Row block: 64 rows for small tensors (<= 4M elements: more blocks in flight), else 256 (fewer
// partials for the finalise).  Measured per rule on B200 (ResNet-18 / ResNet-50 step).
constexpr int kBnRowsBig = 1024;  // large tensors: longer per-thread row loops, 4x fewer partials
inline int64_t bn_big_threshold() {
    static const int64_t v = [] {
        const char *e = std::getenv("CDP_BN_BIG_ELEMS");
        return e ? std::atoll(e) : (int64_t(24) << 20);
    }();
    return v;
}
inline int bn_rows_per_block(int64_t P, int C) {
    return P * C <= (int64_t(4) << 20) ? kBnRowsMin : P * C >= bn_big_threshold() ? kBnRowsBig : kBnRows;
}

template <int KIND, int ROWS>
static __global__ void __launch_bounds__(256) bn_bwd_stats_kernel(const void *__restrict__ g, CTensor mask, int64_t P, int C,
                                                           const void *y, const float *mean, const float *rstd,
                                                           double *partial, const void *y2, const float *mean2,
                                                           const float *rstd2, double *partial2) {
    ptx::griddep_wait();
    ptx::griddep_launch();
    __shared__ float red[3][256 * 4];
    const int C4 = C / 4;
    const int TPR = C4 < 32 ? C4 : 32;
    const int phases = 256 / TPR;
    const int tx = threadIdx.x % TPR, ty = threadIdx.x / TPR;
    const int c = (blockIdx.y * TPR + tx) * 4;
    const int64_t r0 = int64_t(blockIdx.x) * ROWS, r1 = min(P, r0 + ROWS);
    float4 a0 = make_float4(0.f, 0.f, 0.f, 0.f), a1 = a0, b1 = a0;
    const bool active = ty < phases && c < C;
    if (active) {
        const float4 mu = ld_f4(mean, c), rs = ld_f4(rstd, c);
        float4 mu2 = mu, rs2 = rs;
        if (y2) {
            mu2 = ld_f4(mean2, c);
            rs2 = ld_f4(rstd2, c);
        }
#pragma unroll 4
        for (int64_t r = r0 + ty; r < r1; r += phases) {
            const size_t o = size_t(r) * C + c;
            float4 gv = ld_y4<KIND>(g, o);
            if (mask.hi) gv = relu_mask4(gv, ld_c4<KIND>(mask, o));
            const float4 x = ld_y4<KIND>(y, o);
            a0.x += gv.x;
            a0.y += gv.y;
            a0.z += gv.z;
            a0.w += gv.w;
            a1.x = fmaf(gv.x, (x.x - mu.x) * rs.x, a1.x);
            a1.y = fmaf(gv.y, (x.y - mu.y) * rs.y, a1.y);
            a1.z = fmaf(gv.z, (x.z - mu.z) * rs.z, a1.z);
            a1.w = fmaf(gv.w, (x.w - mu.w) * rs.w, a1.w);
            if (y2) {
                const float4 x2 = ld_y4<KIND>(y2, o);
                b1.x = fmaf(gv.x, (x2.x - mu2.x) * rs2.x, b1.x);
                b1.y = fmaf(gv.y, (x2.y - mu2.y) * rs2.y, b1.y);
                b1.z = fmaf(gv.z, (x2.z - mu2.z) * rs2.z, b1.z);
                b1.w = fmaf(gv.w, (x2.w - mu2.w) * rs2.w, b1.w);
            }
        }
    }
    const int slot = threadIdx.x * 4;
    *reinterpret_cast<float4 *>(&red[0][slot]) = a0;
    *reinterpret_cast<float4 *>(&red[1][slot]) = a1;
    *reinterpret_cast<float4 *>(&red[2][slot]) = b1;
    __syncthreads();
    // thread k < TPR*4 combines channel (blockIdx.y*TPR*4 + k) over the phases in order
    const int k = threadIdx.x;
    if (k < TPR * 4) {
        const int cc = blockIdx.y * TPR * 4 + k;
        if (cc < C) {
            const int t = k / 4, j = k % 4;
            double s0 = 0.0, s1 = 0.0, s2 = 0.0;
            for (int ph = 0; ph < phases; ++ph) {
                const int idx = (ph * TPR + t) * 4 + j;
                s0 += double(red[0][idx]);
                s1 += double(red[1][idx]);
                s2 += double(red[2][idx]);
            }
            double *o = partial + (size_t(cc) * gridDim.x + blockIdx.x) * 2;  // [C][blocks][2]
            o[0] = s0;
            o[1] = s1;
            if (partial2) {
                double *o2 = partial2 + (size_t(cc) * gridDim.x + blockIdx.x) * 2;
                o2[0] = s0;
                o2[1] = s2;
            }
        }
    }
}

// bf16 backward statistics, 8 channels (16 bytes) per thread: TPR = min(C/8, 32) threads per row,
// 256/TPR row phases, U rows' loads issued before their arithmetic.  The grid is sized to the GPU
// (two CTAs per SM) and every CTA strides over row chunks of phases * U rows in a fixed order (the
// 4-channel kernel above ran fixed 1024-row blocks: 392 CTAs on the 64-channel ResNet-50 tensors =
// 1.3 waves, 3.4 TB/s).  Same partial layout [C][CTAs][2] (bn_finalize_bwd_kernel over gridDim.x
// partials); phases combined in fixed order in fp64.
template <bool MASK, bool Y2>
static __global__ void __launch_bounds__(256, 2)
    bn_bwd_stats8_kernel(const __nv_bfloat16 *__restrict__ g, const __nv_bfloat16 *__restrict__ mask, int64_t P,
                         int C, const __nv_bfloat16 *__restrict__ y, const float *mean, const float *rstd,
                         double *partial, const __nv_bfloat16 *__restrict__ y2, const float *mean2,
                         const float *rstd2, double *partial2) {
    ptx::griddep_wait();
    ptx::griddep_launch();
    constexpr int NA = Y2 ? 3 : 2;
    constexpr int U = Y2 ? 2 : 4;
    __shared__ __align__(16) float red[NA][256 * 8];
    const int C8 = C / 8;
    const int TPR = C8 < 32 ? C8 : 32;
    const int phases = 256 / TPR;
    const int tx = threadIdx.x % TPR, ty = threadIdx.x / TPR;
    const int c = (blockIdx.y * TPR + tx) * 8;
    const int64_t chunk = int64_t(phases) * U;
    float a0[8], a1[8], b1[8];
#pragma unroll
    for (int k = 0; k < 8; ++k) a0[k] = a1[k] = b1[k] = 0.f;
    if (ty < phases && c < C) {
        const F8 mu = ld_f8(mean, c), rs = ld_f8(rstd, c);
        F8 mu2 = mu, rs2 = rs;
        if constexpr (Y2) {
            mu2 = ld_f8(mean2, c);
            rs2 = ld_f8(rstd2, c);
        }
        const uint4 z4 = make_uint4(0u, 0u, 0u, 0u);
        for (int64_t rb = int64_t(blockIdx.x) * chunk + ty; rb < P; rb += int64_t(gridDim.x) * chunk) {
            uint4 gr[U], yr[U], mr[U], y2r[U];
#pragma unroll
            for (int u = 0; u < U; ++u) {  // rows past the end contribute g = 0
                const int64_t r = rb + int64_t(u) * phases;
                const bool in = r < P;
                const size_t o = size_t(in ? r : rb) * C + c;
                gr[u] = in ? *reinterpret_cast<const uint4 *>(g + o) : z4;
                yr[u] = *reinterpret_cast<const uint4 *>(y + o);
                if constexpr (MASK) mr[u] = *reinterpret_cast<const uint4 *>(mask + o);
                if constexpr (Y2) y2r[u] = *reinterpret_cast<const uint4 *>(y2 + o);
            }
#pragma unroll
            for (int u = 0; u < U; ++u) {
                F8 gv, x;
                bf16x8_to_f8(gr[u], gv);
                bf16x8_to_f8(yr[u], x);
                if constexpr (MASK) {
                    F8 mk;
                    bf16x8_to_f8(mr[u], mk);
#pragma unroll
                    for (int k = 0; k < 8; ++k) gv.v[k] = mk.v[k] > 0.f ? gv.v[k] : 0.f;
                }
#pragma unroll
                for (int k = 0; k < 8; ++k) {
                    a0[k] += gv.v[k];
                    a1[k] = fmaf(gv.v[k], (x.v[k] - mu.v[k]) * rs.v[k], a1[k]);
                }
                if constexpr (Y2) {
                    F8 x2;
                    bf16x8_to_f8(y2r[u], x2);
#pragma unroll
                    for (int k = 0; k < 8; ++k) b1[k] = fmaf(gv.v[k], (x2.v[k] - mu2.v[k]) * rs2.v[k], b1[k]);
                }
            }
        }
    }
    const int slot = threadIdx.x * 8;
    *reinterpret_cast<float4 *>(&red[0][slot]) = make_float4(a0[0], a0[1], a0[2], a0[3]);
    *reinterpret_cast<float4 *>(&red[0][slot + 4]) = make_float4(a0[4], a0[5], a0[6], a0[7]);
    *reinterpret_cast<float4 *>(&red[1][slot]) = make_float4(a1[0], a1[1], a1[2], a1[3]);
    *reinterpret_cast<float4 *>(&red[1][slot + 4]) = make_float4(a1[4], a1[5], a1[6], a1[7]);
    if constexpr (Y2) {
        *reinterpret_cast<float4 *>(&red[NA - 1][slot]) = make_float4(b1[0], b1[1], b1[2], b1[3]);
        *reinterpret_cast<float4 *>(&red[NA - 1][slot + 4]) = make_float4(b1[4], b1[5], b1[6], b1[7]);
    }
    __syncthreads();
    // thread k < TPR*8 combines channel (blockIdx.y*TPR*8 + k) over the phases in order
    const int k = threadIdx.x;
    if (k < TPR * 8) {
        const int cc = blockIdx.y * TPR * 8 + k;
        if (cc < C) {
            double s0 = 0.0, s1 = 0.0, s2 = 0.0;
            for (int ph = 0; ph < phases; ++ph) {
                const int idx = ph * TPR * 8 + k;
                s0 += double(red[0][idx]);
                s1 += double(red[1][idx]);
                if constexpr (Y2) s2 += double(red[NA - 1][idx]);
            }
            double *o = partial + (size_t(cc) * gridDim.x + blockIdx.x) * 2;  // [C][blocks][2]
            o[0] = s0;
            o[1] = s1;
            if constexpr (Y2) {
                double *o2 = partial2 + (size_t(cc) * gridDim.x + blockIdx.x) * 2;
                o2[0] = s0;
                o2[1] = s2;
            }
        }
    }
}

// Backward finalise: dbeta = sum g', dgamma = sum g' xhat over the row blocks in order.
static __global__ void bn_finalize_bwd_kernel(const double *__restrict__ partial, int nblk, int C, float *dbeta,
                                       float *dgamma) {
    ptx::griddep_wait();
    ptx::griddep_launch();
    const int c = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const int lane = threadIdx.x & 31;
    if (c >= C) return;
    double s0 = 0.0, s1 = 0.0;
    const double2 *pc = reinterpret_cast<const double2 *>(partial) + size_t(c) * nblk;  // [C][blocks]
    for (int t = lane; t < nblk; t += 32) {
        const double2 v = pc[t];
        s0 += v.x;
        s1 += v.y;
    }
#pragma unroll
    for (int o = 16; o; o >>= 1) {
        s0 += __shfl_xor_sync(0xffffffffu, s0, o);
        s1 += __shfl_xor_sync(0xffffffffu, s1, o);
    }
    if (lane == 0) {
        dbeta[c] = float(s0);
        dgamma[c] = float(s1);
    }
}

// Backward through BN (+ReLU mask): dx = gamma * rstd * (g' - dbeta/P - xhat * dgamma/P)
// in compute format (the conv's output gradient, a GEMM operand).  bf16 mode: per channel
// the thread keeps mean, k1 = gamma * rstd, k2 = dbeta / P, k3 = rstd * dgamma / P and
// computes dx = k1 * (g' - k2 - (x - mean) * k3) (32 coefficient registers instead of 40);
// fp32 (parity) mode keeps the restatement's evaluation order.
template <int KIND>
struct BnBwd {
    F8 mu, k1, k2, k3, k4;  // KIND 1: k1 = rstd, k2 = gamma, k3 = dbeta, k4 = dgamma
    float inv;
    __device__ __forceinline__ void load(const float *mean, const float *rstd, const float *gamma,
                                         const float *dbeta, const float *dgamma, int c) {
        mu = ld_f8(mean, c);
        if constexpr (KIND == 0) {
            const F8 rs = ld_f8(rstd, c), ga = ld_f8(gamma, c), db = ld_f8(dbeta, c), dg = ld_f8(dgamma, c);
#pragma unroll
            for (int k = 0; k < 8; ++k) {
                k1.v[k] = ga.v[k] * rs.v[k];
                k2.v[k] = db.v[k] * inv;
                k3.v[k] = rs.v[k] * (dg.v[k] * inv);
            }
        } else {
            k1 = ld_f8(rstd, c);
            k2 = ld_f8(gamma, c);
            k3 = ld_f8(dbeta, c);
            k4 = ld_f8(dgamma, c);
        }
    }
    __device__ __forceinline__ float operator()(float g, float x, int k) const {
        if constexpr (KIND == 0)
            return k1.v[k] * (g - k2.v[k] - (x - mu.v[k]) * k3.v[k]);
        else
            return k2.v[k] * k1.v[k] * (g - k3.v[k] * inv - ((x - mu.v[k]) * k1.v[k]) * k4.v[k] * inv);
    }
};

template <int KIND, bool MASK>
static __global__ void __launch_bounds__(256) bn_bwd_apply_kernel(const void *__restrict__ g, CTensor mask,
                                                                  const void *__restrict__ y, int64_t P, int C,
                                                                  const float *mean, const float *rstd,
                                                                  const float *gamma, const float *dbeta,
                                                                  const float *dgamma, CTensor dx) {
    ptx::griddep_wait();
    ptx::griddep_launch();
    const int C8 = C / 8;
    const int64_t n = P * C8;
    const int64_t stride = int64_t(gridDim.x) * blockDim.x;
    const bool fixed = stride % C8 == 0;  // the thread's channels never change (parameters loaded once)
    int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x;
    BnBwd<KIND> f;
    f.inv = 1.f / float(P);
    f.load(mean, rstd, gamma, dbeta, dgamma, int(i % C8) * 8);
    if constexpr (KIND == 0) if (fixed) {  // U vectors' loads before any store (see bn_apply_kernel)
        constexpr int U = MASK ? 2 : 4;
        const uint4 *gp = static_cast<const uint4 *>(g), *yp = static_cast<const uint4 *>(y);
        const uint4 *mp = static_cast<const uint4 *>(mask.hi);
        for (; i < n; i += stride * U) {
            uint4 a[U], b[U], m[U];
#pragma unroll
            for (int u = 0; u < U; ++u) {
                const int64_t j = i + u * stride;
                if (j < n) {
                    a[u] = gp[j];
                    b[u] = yp[j];
                    if constexpr (MASK) m[u] = mp[j];
                }
            }
#pragma unroll
            for (int u = 0; u < U; ++u) {
                const int64_t j = i + u * stride;
                if (j >= n) break;
                F8 gv, x, mk, d;
                bf16x8_to_f8(a[u], gv);
                bf16x8_to_f8(b[u], x);
                if constexpr (MASK) bf16x8_to_f8(m[u], mk);
#pragma unroll
                for (int k = 0; k < 8; ++k) {
                    const float gk = (MASK && !(mk.v[k] > 0.f)) ? 0.f : gv.v[k];
                    d.v[k] = f(gk, x.v[k], k);
                }
                static_cast<uint4 *>(dx.hi)[j] = f8_to_bf16x8(d);
            }
        }
        return;
    }
#pragma unroll 2
    for (; i < n; i += stride) {
        if (!fixed) f.load(mean, rstd, gamma, dbeta, dgamma, int(i % C8) * 8);
        const size_t o = size_t(i) * 8;
        const F8 gv = ld_y8<KIND>(g, o);
        const F8 x = ld_y8<KIND>(y, o);
        F8 mk;
        if constexpr (MASK) mk = ld_c8<KIND>(mask, o);
        F8 d;
#pragma unroll
        for (int k = 0; k < 8; ++k) {
            const float gk = (MASK && !(mk.v[k] > 0.f)) ? 0.f : gv.v[k];
            d.v[k] = f(gk, x.v[k], k);
        }
        st_c8<KIND>(dx, o, d);
    }
}

// ---------------------------------------------------------------------------
// Max pool 3x3 / stride 2 / pad 1 (ImageNet stem).  Forward keeps the winning
// tap (first maximum in (r, s) order) per output element; backward routes each
// window's gradient to its tap, owner-computes (below), deterministic.
// 8 channels per thread: 16-byte activation / gradient accesses, 8-byte tap records.
template <int KIND>
static __global__ void maxpool_fwd_kernel(CTensor in, int B, int H, int W, int C, int Ho, int Wo, CTensor out,
                                   uint8_t *arg) {
    ptx::griddep_wait();
    ptx::griddep_launch();
    const int C8 = C / 8;
    const int64_t n = int64_t(B) * Ho * Wo * C8;
    for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < n; i += int64_t(gridDim.x) * blockDim.x) {
        const int c = int(i % C8) * 8;
        const int p = int(i / C8);
        const int wo = p % Wo, t = p / Wo, ho = t % Ho, b = t / Ho;
        F8 best;
        uint8_t bt[8];
#pragma unroll
        for (int j = 0; j < 8; ++j) {
            best.v[j] = -INFINITY;
            bt[j] = 0;
        }
        if constexpr (KIND == 0) {  // the nine window loads issued before any compare (latency-bound otherwise)
            uint4 raw[9];
            bool ok[9];
#pragma unroll
            for (int k = 0; k < 9; ++k) {
                const int h = ho * 2 - 1 + k / 3, w = wo * 2 - 1 + k % 3;
                ok[k] = h >= 0 && h < H && w >= 0 && w < W;
                raw[k] = ok[k] ? *reinterpret_cast<const uint4 *>(static_cast<const __nv_bfloat16 *>(in.hi) +
                                                                  ((size_t(b) * H + h) * W + w) * in.ld + c)
                               : make_uint4(0, 0, 0, 0);
            }
#pragma unroll
            for (int k = 0; k < 9; ++k) {
                if (!ok[k]) continue;
                F8 v;
                bf16x8_to_f8(raw[k], v);
#pragma unroll
                for (int j = 0; j < 8; ++j)
                    if (v.v[j] > best.v[j]) {
                        best.v[j] = v.v[j];
                        bt[j] = uint8_t(k);
                    }
            }
        } else {
            for (int r = 0; r < 3; ++r) {
                const int h = ho * 2 - 1 + r;
                if (h < 0 || h >= H) continue;
                for (int s = 0; s < 3; ++s) {
                    const int w = wo * 2 - 1 + s;
                    if (w < 0 || w >= W) continue;
                    const F8 v = ld_c8<KIND>(in, ((size_t(b) * H + h) * W + w) * in.ld + c);
#pragma unroll
                    for (int j = 0; j < 8; ++j)
                        if (v.v[j] > best.v[j]) {
                            best.v[j] = v.v[j];
                            bt[j] = uint8_t(r * 3 + s);
                        }
                }
            }
        }
        st_c8<KIND>(out, size_t(p) * out.ld + c, best);
        uint2 packed;
        packed.x = uint32_t(bt[0]) | uint32_t(bt[1]) << 8 | uint32_t(bt[2]) << 16 | uint32_t(bt[3]) << 24;
        packed.y = uint32_t(bt[4]) | uint32_t(bt[5]) << 8 | uint32_t(bt[6]) << 16 | uint32_t(bt[7]) << 24;
        *reinterpret_cast<uint2 *>(arg + size_t(p) * C + c) = packed;
    }
}

// Max-pool backward by owner: a thread takes the 2x2 input pixels (2ho .. 2ho+1, 2wo .. 2wo+1) of one
// output position and 8 channels, reads the (at most) four windows that can route into them (ho, ho+1) x
// (wo, wo+1) once each, and writes the four pixels - 4 window reads per 4 pixels instead of the gather's 9,
// and the index arithmetic once per 4 pixels (the gather kernel ran at 1.3 TB/s).  Windows are added in
// (ho', wo') order: deterministic.
template <int KIND>
static __global__ void __launch_bounds__(256) maxpool_bwd_owner_kernel(const void *__restrict__ gout,
                                                                       const uint8_t *__restrict__ arg, int B, int H,
                                                                       int W, int C, int Ho, int Wo, void *gin) {
    ptx::griddep_wait();
    ptx::griddep_launch();
    const int C8 = C / 8;
    const int64_t n = int64_t(B) * Ho * Wo * C8;
    for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < n; i += int64_t(gridDim.x) * blockDim.x) {
        const int c = int(i % C8) * 8;
        const int q = int(i / C8);
        const int wo = q % Wo, t = q / Wo, ho = t % Ho, b = t / Ho;
        F8 acc[2][2];
#pragma unroll
        for (int a = 0; a < 2; ++a)
#pragma unroll
            for (int e = 0; e < 2; ++e)
#pragma unroll
                for (int j = 0; j < 8; ++j) acc[a][e].v[j] = 0.f;
#pragma unroll
        for (int dh = 0; dh < 2; ++dh) {
            if (ho + dh >= Ho) continue;
#pragma unroll
            for (int dw = 0; dw < 2; ++dw) {
                if (wo + dw >= Wo) continue;
                const size_t o = ((size_t(b) * Ho + ho + dh) * Wo + wo + dw) * C + c;
                const uint2 a = __ldg(reinterpret_cast<const uint2 *>(arg + o));
                const F8 g = ld_y8<KIND>(gout, o);
#pragma unroll
                for (int j = 0; j < 8; ++j) {
                    const int tap = int(((j < 4 ? a.x : a.y) >> (8 * (j & 3))) & 0xffu);
                    const int r = tap / 3, s = tap - 3 * (tap / 3);
                    // window (ho + dh) covers input rows 2(ho + dh) - 1 + r: owned row offset 2 dh - 1 + r
                    const int orow = 2 * dh - 1 + r, ocol = 2 * dw - 1 + s;
                    if (orow == 0 && ocol == 0) acc[0][0].v[j] += g.v[j];
                    else if (orow == 0 && ocol == 1) acc[0][1].v[j] += g.v[j];
                    else if (orow == 1 && ocol == 0) acc[1][0].v[j] += g.v[j];
                    else if (orow == 1 && ocol == 1) acc[1][1].v[j] += g.v[j];
                }
            }
        }
#pragma unroll
        for (int a = 0; a < 2; ++a) {
            const int h = 2 * ho + a;
            if (h >= H) continue;
#pragma unroll
            for (int e = 0; e < 2; ++e) {
                const int w = 2 * wo + e;
                if (w < W) st_y8<KIND>(gin, ((size_t(b) * H + h) * W + w) * C + c, acc[a][e]);
            }
        }
    }
}

// Global average pool: act [B*HW][ld] -> pooled [B][C+1] (ones column at C for the fc bias).
template <int KIND>
static __global__ void avgpool_kernel(CTensor act, int B, int HW, int C, CTensor pooled) {
    ptx::griddep_wait();
    ptx::griddep_launch();
    const int b = blockIdx.x;
    for (int c = threadIdx.x; c <= C; c += blockDim.x) {
        float s = 0.f;
        if (c < C) {
            for (int k = 0; k < HW; ++k) s += Fmt<KIND>::load(act.hi, act.lo, (size_t(b) * HW + k) * act.ld + c);
            s /= float(HW);
        } else {
            s = 1.f;
        }
        Fmt<KIND>::store(pooled.hi, pooled.lo, size_t(b) * pooled.ld + c, s);
    }
}

// d act[b, k, c] = dpooled[b][c] / HW (Y format), 4 channels per thread.
template <int KIND>
static __global__ void avgpool_backward_kernel(const float *dp, int ldp, int B, int HW, int C, void *g,
                                               CTensor mask) {
    ptx::griddep_wait();
    ptx::griddep_launch();
    const int C4 = C / 4;
    const int64_t n = int64_t(B) * HW * C4;
    const float inv = 1.f / float(HW);
    for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < n; i += int64_t(gridDim.x) * blockDim.x) {
        const int c = int(i % C4) * 4;
        const int64_t r = i / C4;
        const float *s = dp + (r / HW) * ldp + c;
        float4 v = make_float4(s[0] * inv, s[1] * inv, s[2] * inv, s[3] * inv);
        if (mask.hi) v = relu_mask4(v, ld_c4<KIND>(mask, size_t(r) * C + c));  // the last block's ReLU
        st_y4<KIND>(g, size_t(r) * C + c, v);
    }
}

// Softmax cross-entropy for many classes (ImageNet heads): one CTA per sample,
// fixed-tree block reductions; per-sample losses summed in ascending sample
// order by loss_sum_kernel (ref _kernels.pyx:80-100 semantics).
template <int KIND>
static __global__ void __launch_bounds__(256) xent_rows_kernel(const float *__restrict__ z, int B, int C, const int *perm,
                                                        const int *labels, CTensor dz, double *loss_rows) {
    ptx::griddep_wait();
    ptx::griddep_launch();
    __shared__ float red[256];
    const int s = blockIdx.x, tid = threadIdx.x;
    const float *zr = z + size_t(s) * C;
    float mx = -INFINITY;
    for (int o = tid; o < C; o += blockDim.x) mx = fmaxf(mx, zr[o]);
    red[tid] = mx;
    __syncthreads();
    for (int k = 128; k; k >>= 1) {
        if (tid < k) red[tid] = fmaxf(red[tid], red[tid + k]);
        __syncthreads();
    }
    mx = red[0];
    __syncthreads();
    float se = 0.f;
    for (int o = tid; o < C; o += blockDim.x) se += expf(zr[o] - mx);
    red[tid] = se;
    __syncthreads();
    for (int k = 128; k; k >>= 1) {
        if (tid < k) red[tid] += red[tid + k];
        __syncthreads();
    }
    se = red[0];
    const int lab = labels[perm[s]];
    for (int o = tid; o < C; o += blockDim.x) {
        const float pz = __fdiv_rn(expf(zr[o] - mx), se);
        Fmt<KIND>::store(dz.hi, dz.lo, size_t(s) * dz.ld + o, __fdiv_rn(pz - (o == lab ? 1.f : 0.f), float(B)));
        if (o == lab) loss_rows[s] = double(mx) - double(zr[o]) + log(double(se));  // finite when pz underflows
    }
}

static __global__ void loss_sum_kernel(const double *rows, int B, double *loss_out, unsigned *loss_flag) {
    ptx::griddep_wait();
    ptx::griddep_launch();
    double acc = 0.0;
    for (int k = 0; k < B; ++k) acc += rows[k];
    acc /= B;
    *loss_out = acc;
    if (!isfinite(acc)) atomicOr(loss_flag, 1u);
}

// Data gradient of the classifier: plain fp32 store of (W . dZ^T)[k, s] as dpooled[s][k].
struct EpiDgradLinear {
    struct Params {
        float *out;
        int ld;
    };
    struct State {};
    __device__ static void begin(const Params &, int, State &) {}
    __device__ static void apply(const Params &p, int m, int n0, const float (&v)[32], int M, int N, State &) {
        if (m >= M) return;
#pragma unroll
        for (int i = 0; i < 32; ++i)
            if (n0 + i < N) p.out[size_t(n0 + i) * p.ld + m] = v[i];
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

// DP all-reduce baseline: update of one parameter tensor from the collective-summed
// gradient (p.s_in), the reference's update arithmetic (engine.py:102-109) in fp32,
// repacking the GEMM compute copy ([rows][ld], `cols` per row) when the tensor has one.
template <int KIND>
static __global__ void update_flat_kernel(HopParams p, int64_t n, int cols) {
    ptx::griddep_wait();
    ptx::griddep_launch();
    const float lr = *p.lr;
    bool bad = false;
    for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < n; i += int64_t(gridDim.x) * blockDim.x) {
        const int64_t idx = p.base + i;
        float v = p.momentum != 0.f ? p.vel[idx] : 0.f;
        const float nt = sgd_update(p, p.s_in[idx], p.theta_cur[idx], v, lr);
        if (p.momentum != 0.f) p.vel[idx] = v;
        if (!isfinite(nt)) bad = true;
        p.theta_new[idx] = nt;
        if (p.wc_new.hi) Fmt<KIND>::store(p.wc_new.hi, p.wc_new.lo, size_t(i / cols) * p.wc_new.ld + i % cols, nt);
    }
    if (bad) atomicOr(p.upd_flags, 1u << ((p.stage - 1) & 31));
}

// The pre-hop waits of a weight hop (EpiWgrad::pre) in a one-CTA kernel ahead
// of the GEMM, so that a GEMM grid never occupies SMs while it waits for a peer
// (no dependent launch is triggered before the waits are over).
static __global__ void hop_wait_kernel(HopParams p) { EpiWgrad<0>::pre(p, threadIdx.x, true); }

// Hop / update of a small parameter vector (batch-norm gamma|beta, gradient
// g[0..n) = [dgamma | dbeta] in the parameter order) with the same modes and
// ring protocol as the weight-gradient epilogue.  One CTA of 128 threads.
static __global__ void vector_hop_kernel(HopParams p, const float *dgamma, const float *dbeta, int C) {
    ptx::griddep_wait();
    ptx::griddep_launch();
    EpiWgrad<0>::pre(p, threadIdx.x);
    bool bg = false, bu = false;
    for (int i = threadIdx.x; i < 2 * C; i += blockDim.x) {
        const float g = i < C ? dgamma[i] : dbeta[i - C];
        hop_elem<0>(p, p.base + i, g, 0, false, bg, bu);
    }
    if (bg) atomicOr(p.grad_flags, 1u << ((p.stage - 1) & 31));
    if (bu) atomicOr(p.upd_flags, 1u << ((p.stage - 1) & 31));
    EpiWgrad<0>::post(p, threadIdx.x, 1);
}

}  // namespace cdp
