// Convolutional-network layer kernels for the ResNet configs (BASELINE
// configs[1..2,4]).  Convolutions are tcgen05 GEMMs (gemm_tc_kernel): implicit
// (TMA-gathered NHWC boxes, MODE 1-3) for every conv whose input channels fill a
// 128-byte chunk, a plain GEMM for 1x1 stride-1 convs, and an explicit im2col
// only for the 3-channel stem.  Batch norm runs in training mode (per
// micro-batch statistics) with fixed-order reductions: the forward statistics
// come out of the conv GEMM's epilogue (per M tile), the backward ones from a
// row-blocked partial kernel; both are finalised in fp64 in a fixed order.
//
// Storage: activations in the GEMM compute format (bf16, or fp32 hi/lo for the
// 3xTF32 mode); conv outputs y in "Y format" (bf16 / fp32); gradients flowing
// between layers fp32.  All elementwise kernels move 4 channels per thread.
#pragma once
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

// ---------------------------------------------------------------------------
// Stem: gather the micro-batch's images (fp32 NHWC dataset rows, C = 3) and
// im2col them in one pass: cols[p][k], k = (r*S + s)*C + c, zero padding and
// zero columns K..ld-1.  The cols matrix is the stem's activation record.
template <int KIND>
__global__ void stem_im2col_kernel(const float *__restrict__ data, const int *perm, int H, int W, int C, int R, int S,
                                   int stride, int pad, int Ho, int Wo, int64_t P, CTensor cols) {
    ptx::griddep_wait();
    ptx::griddep_launch();
    const int K = R * S * C;
    const int64_t n = P * cols.ld;
    for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < n; i += int64_t(gridDim.x) * blockDim.x) {
        const int k = int(i % cols.ld);
        const int64_t p = i / cols.ld;
        float v = 0.f;
        if (k < K) {
            const int c = k % C, rs = k / C, s = rs % S, r = rs / S;
            const int wo = int(p % Wo), ho = int((p / Wo) % Ho), b = int(p / (int64_t(Wo) * Ho));
            const int h = ho * stride - pad + r, w = wo * stride - pad + s;
            if (h >= 0 && h < H && w >= 0 && w < W) v = data[((size_t(perm[b]) * H + h) * W + w) * C + c];
        }
        Fmt<KIND>::store(cols.hi, cols.lo, size_t(i), v);
    }
}

// col2im (deterministic gather) for the convs whose data gradient is an explicit
// GEMM into im2col space (stride 2): dx[b,h,w,c] = sum over (r, s) ascending of
// dcols[(b, ho, wo), (r, s, c)] with h = ho*stride - pad + r.  4 channels per thread.
__global__ void col2im_kernel(const float *__restrict__ dcols, int ldc, int B, int H, int W, int C, int R, int S,
                              int stride, int pad, int Ho, int Wo, float *dx) {
    ptx::griddep_wait();
    ptx::griddep_launch();
    const int C4 = C / 4;
    const int64_t n = int64_t(B) * H * W * C4;
    for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < n; i += int64_t(gridDim.x) * blockDim.x) {
        const int c = int(i % C4) * 4;
        const int64_t pix = i / C4;
        const int w = int(pix % W), h = int((pix / W) % H), b = int(pix / (int64_t(W) * H));
        float4 acc = make_float4(0.f, 0.f, 0.f, 0.f);
        for (int r = 0; r < R; ++r) {
            const int hh = h + pad - r;
            if (hh < 0 || hh % stride) continue;
            const int ho = hh / stride;
            if (ho >= Ho) continue;
            for (int s = 0; s < S; ++s) {
                const int ww = w + pad - s;
                if (ww < 0 || ww % stride) continue;
                const int wo = ww / stride;
                if (wo >= Wo) continue;
                const float4 v = ld_f4(dcols, (size_t(b) * Ho * Wo + size_t(ho) * Wo + wo) * ldc + (r * S + s) * C + c);
                acc.x += v.x;
                acc.y += v.y;
                acc.z += v.z;
                acc.w += v.w;
            }
        }
        st_f4(dx, size_t(pix) * C + c, acc);
    }
}

// ---------------------------------------------------------------------------
// Conv GEMM epilogue (tile form): the 128 x BN fp32 tile is in shared memory.
// Stores the rows that map to pixels (boxed tiles: conv_box_row; plain tiles:
// m0 + r) either in Y format (forward conv output) or fp32 (data gradient),
// and, when stats != null, the tile's per-channel (sum, sum of squares) over its
// valid rows in ascending row order -> stats[tile][N][2] (BN forward statistics).
template <int KIND>
struct EpiConvOut {
    struct Params {
        void *out;
        int ld;
        int out_f32;   // 1: fp32 rows (gradients); 0: Y format
        float *stats;  // null: no statistics
        int boxed;
        ConvGeom g;
    };
    static constexpr bool kTile = true;
    static constexpr int kStages = 4;
    template <int BN>
    static constexpr int pf_bytes() { return 0; }
    struct State {};
    __device__ static void begin(const Params &, int, State &) {}
    __device__ static void apply(const Params &, int, int, const float (&)[32], int, int, State &) {}
    __device__ static void finish(const Params &, int, int, State &) {}
    __device__ static void extra(const Params &, int, int) {}
    template <int BN>
    __device__ static void prefetch(const Params &, float *, int, int, int, int, int, int) {}
    __device__ static void pre(const Params &, int) {}
    __device__ static void post(const Params &, int, unsigned) {}

    template <int BN>
    __device__ static void tile(const Params &p, const float *st, int lds, const float *, int m0, int n0, int M, int N,
                                int tid, int nth) {
        int *rowm = const_cast<int *>(reinterpret_cast<const int *>(st + 128 * lds));
        for (int r = tid; r < 128; r += nth) {
            int m = p.boxed ? conv_box_row(p.g, blockIdx.x, r) : m0 + r;
            rowm[r] = (m >= 0 && m < M) ? m : -1;
        }
        __syncthreads();
        constexpr int C4 = BN / 4;
        for (int e = tid; e < 128 * C4; e += nth) {
            const int r = e / C4, c = (e % C4) * 4;
            const int m = rowm[r];
            if (m < 0 || n0 + c >= N) continue;
            const float4 v = *reinterpret_cast<const float4 *>(st + r * lds + c);
            const size_t o = size_t(m) * p.ld + n0 + c;
            if (p.out_f32)
                st_f4(static_cast<float *>(p.out), o, v);
            else
                st_y4<KIND>(p.out, o, v);
        }
        if (p.stats) {
            for (int c = tid; c < BN; c += nth) {
                if (n0 + c >= N) continue;
                float s = 0.f, q = 0.f;
                for (int r = 0; r < 128; ++r) {
                    if (rowm[r] < 0) continue;
                    const float v = st[r * lds + c];
                    s += v;
                    q = fmaf(v, v, q);
                }
                float *o = p.stats + (size_t(blockIdx.x) * N + n0 + c) * 2;
                o[0] = s;
                o[1] = q;
            }
        }
    }
};

// Weight gradient of a conv fused with its hop / update: EpiWgrad with a deeper
// operand ring (K = pixels is long).
template <int KIND>
struct EpiWgradConv : EpiWgrad<KIND> {
    static constexpr int kStages = 4;
};

// ---------------------------------------------------------------------------
// Batch norm (training mode).
// Forward finalise: per channel, the per-tile (sum, sum sq) in tile order (fp64)
// -> mean, rstd (biased variance, eps).  One warp per channel, lanes take tiles
// lane, lane+32, ... then a fixed xor-tree: deterministic.
__global__ void bn_finalize_fwd_kernel(const float *__restrict__ stats, int tiles, int C, int64_t P, float eps,
                                       float *mean, float *rstd) {
    ptx::griddep_wait();
    ptx::griddep_launch();
    const int c = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const int lane = threadIdx.x & 31;
    if (c >= C) return;
    double s0 = 0.0, s1 = 0.0;
    for (int t = lane; t < tiles; t += 32) {
        s0 += double(stats[(size_t(t) * C + c) * 2]);
        s1 += double(stats[(size_t(t) * C + c) * 2 + 1]);
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

template <int KIND>
__global__ void bn_apply_kernel(const void *__restrict__ y, int64_t P, int C, const float *mean, const float *rstd,
                                const float *gamma, const float *beta, BnResidual res, int relu, CTensor out) {
    ptx::griddep_wait();
    ptx::griddep_launch();
    const int C4 = C / 4;
    const int64_t n = P * C4;
    for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < n; i += int64_t(gridDim.x) * blockDim.x) {
        const int c = int(i % C4) * 4;
        const size_t o = size_t(i) * 4;
        const float4 x = ld_y4<KIND>(y, o);
        const float4 mu = ld_f4(mean, c), rs = ld_f4(rstd, c), ga = ld_f4(gamma, c), be = ld_f4(beta, c);
        float4 v = make_float4(ga.x * ((x.x - mu.x) * rs.x) + be.x, ga.y * ((x.y - mu.y) * rs.y) + be.y,
                               ga.z * ((x.z - mu.z) * rs.z) + be.z, ga.w * ((x.w - mu.w) * rs.w) + be.w);
        if (res.act.hi) {
            const float4 a = ld_c4<KIND>(res.act, o);
            v.x += a.x;
            v.y += a.y;
            v.z += a.z;
            v.w += a.w;
        }
        if (res.y) {
            const float4 x2 = ld_y4<KIND>(res.y, o);
            const float4 m2 = ld_f4(res.mean, c), r2 = ld_f4(res.rstd, c), g2 = ld_f4(res.gamma, c),
                         b2 = ld_f4(res.beta, c);
            v.x += g2.x * ((x2.x - m2.x) * r2.x) + b2.x;
            v.y += g2.y * ((x2.y - m2.y) * r2.y) + b2.y;
            v.z += g2.z * ((x2.z - m2.z) * r2.z) + b2.z;
            v.w += g2.w * ((x2.w - m2.w) * r2.w) + b2.w;
        }
        if (relu) v = make_float4(fmaxf(v.x, 0.f), fmaxf(v.y, 0.f), fmaxf(v.z, 0.f), fmaxf(v.w, 0.f));
        store_wc4<KIND>(out, o, v);
    }
}

// Backward statistics: per row block (kBnRows rows), per channel,
// (sum g', sum g' * xhat) with g' = g masked by (act > 0) when mask != null.
// TPR threads per row (4 channels each), 256/TPR row phases; the phases are
// combined in fixed order in fp64 -> partial[blk][C][2].  A second conv output
// (projection shortcut: same g', own y / stats) gives partial2.
constexpr int kBnRows = 256;

template <int KIND>
__global__ void __launch_bounds__(256) bn_bwd_stats_kernel(const float *__restrict__ g, CTensor mask, int64_t P, int C,
                                                           const void *y, const float *mean, const float *rstd,
                                                           double *partial, const void *y2, const float *mean2,
                                                           const float *rstd2, double *partial2) {
    ptx::griddep_wait();
    ptx::griddep_launch();
    __shared__ float red[4][256 * 4];
    const int C4 = C / 4;
    const int TPR = C4 < 32 ? C4 : 32;
    const int phases = 256 / TPR;
    const int tx = threadIdx.x % TPR, ty = threadIdx.x / TPR;
    const int c = (blockIdx.y * TPR + tx) * 4;
    const int64_t r0 = int64_t(blockIdx.x) * kBnRows, r1 = min(P, r0 + kBnRows);
    float4 a0 = make_float4(0.f, 0.f, 0.f, 0.f), a1 = a0, b1 = a0;
    const bool active = ty < phases && c < C;
    if (active) {
        const float4 mu = ld_f4(mean, c), rs = ld_f4(rstd, c);
        float4 mu2 = mu, rs2 = rs;
        if (y2) {
            mu2 = ld_f4(mean2, c);
            rs2 = ld_f4(rstd2, c);
        }
        for (int64_t r = r0 + ty; r < r1; r += phases) {
            const size_t o = size_t(r) * C + c;
            float4 gv = ld_f4(g, o);
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
            double *o = partial + (size_t(blockIdx.x) * C + cc) * 2;
            o[0] = s0;
            o[1] = s1;
            if (partial2) {
                double *o2 = partial2 + (size_t(blockIdx.x) * C + cc) * 2;
                o2[0] = s0;
                o2[1] = s2;
            }
        }
    }
}

// Backward finalise: dbeta = sum g', dgamma = sum g' xhat over the row blocks in order.
__global__ void bn_finalize_bwd_kernel(const double *__restrict__ partial, int nblk, int C, float *dbeta,
                                       float *dgamma) {
    ptx::griddep_wait();
    ptx::griddep_launch();
    const int c = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const int lane = threadIdx.x & 31;
    if (c >= C) return;
    double s0 = 0.0, s1 = 0.0;
    for (int t = lane; t < nblk; t += 32) {
        s0 += partial[(size_t(t) * C + c) * 2];
        s1 += partial[(size_t(t) * C + c) * 2 + 1];
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
// in compute format (the conv's output gradient, a GEMM operand).
template <int KIND>
__global__ void bn_bwd_apply_kernel(const float *__restrict__ g, CTensor mask, const void *__restrict__ y, int64_t P,
                                    int C, const float *mean, const float *rstd, const float *gamma,
                                    const float *dbeta, const float *dgamma, CTensor dx) {
    ptx::griddep_wait();
    ptx::griddep_launch();
    const int C4 = C / 4;
    const int64_t n = P * C4;
    const float inv = 1.f / float(P);
    for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < n; i += int64_t(gridDim.x) * blockDim.x) {
        const int c = int(i % C4) * 4;
        const size_t o = size_t(i) * 4;
        float4 gv = ld_f4(g, o);
        if (mask.hi) gv = relu_mask4(gv, ld_c4<KIND>(mask, o));
        const float4 x = ld_y4<KIND>(y, o);
        const float4 mu = ld_f4(mean, c), rs = ld_f4(rstd, c), ga = ld_f4(gamma, c), db = ld_f4(dbeta, c),
                     dg = ld_f4(dgamma, c);
        float4 d;
        d.x = ga.x * rs.x * (gv.x - db.x * inv - ((x.x - mu.x) * rs.x) * dg.x * inv);
        d.y = ga.y * rs.y * (gv.y - db.y * inv - ((x.y - mu.y) * rs.y) * dg.y * inv);
        d.z = ga.z * rs.z * (gv.z - db.z * inv - ((x.z - mu.z) * rs.z) * dg.z * inv);
        d.w = ga.w * rs.w * (gv.w - db.w * inv - ((x.w - mu.w) * rs.w) * dg.w * inv);
        store_wc4<KIND>(dx, o, d);
    }
}

// out = a + b (fp32 [P][C]), b masked by (mask > 0) when mask != null.
template <int KIND>
__global__ void add_kernel(const float *a, const float *b, int64_t P, int C, CTensor mask_b, float *out) {
    ptx::griddep_wait();
    ptx::griddep_launch();
    const int64_t n = P * C / 4;
    for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < n; i += int64_t(gridDim.x) * blockDim.x) {
        const size_t o = size_t(i) * 4;
        float4 vb = ld_f4(b, o);
        if (mask_b.hi) vb = relu_mask4(vb, ld_c4<KIND>(mask_b, o));
        const float4 va = ld_f4(a, o);
        st_f4(out, o, make_float4(va.x + vb.x, va.y + vb.y, va.z + vb.z, va.w + vb.w));
    }
}

// ---------------------------------------------------------------------------
// Max pool 3x3 / stride 2 / pad 1 (ImageNet stem).  Forward keeps the winning
// tap (first maximum in (r, s) order) per output element; backward is a
// deterministic gather over the (at most 4) windows containing an input pixel.
template <int KIND>
__global__ void maxpool_fwd_kernel(CTensor in, int B, int H, int W, int C, int Ho, int Wo, CTensor out,
                                   uint8_t *arg) {
    ptx::griddep_wait();
    ptx::griddep_launch();
    const int64_t n = int64_t(B) * Ho * Wo * C;
    for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < n; i += int64_t(gridDim.x) * blockDim.x) {
        const int c = int(i % C);
        const int64_t p = i / C;
        const int wo = int(p % Wo), ho = int((p / Wo) % Ho), b = int(p / (int64_t(Wo) * Ho));
        float best = -INFINITY;
        int bt = 0;
        for (int r = 0; r < 3; ++r) {
            const int h = ho * 2 - 1 + r;
            if (h < 0 || h >= H) continue;
            for (int s = 0; s < 3; ++s) {
                const int w = wo * 2 - 1 + s;
                if (w < 0 || w >= W) continue;
                const float v = Fmt<KIND>::load(in.hi, in.lo, ((size_t(b) * H + h) * W + w) * in.ld + c);
                if (v > best) {
                    best = v;
                    bt = r * 3 + s;
                }
            }
        }
        Fmt<KIND>::store(out.hi, out.lo, size_t(p) * out.ld + c, best);
        arg[i] = uint8_t(bt);
    }
}

__global__ void maxpool_bwd_kernel(const float *__restrict__ gout, const uint8_t *__restrict__ arg, int B, int H, int W,
                                   int C, int Ho, int Wo, float *gin) {
    ptx::griddep_wait();
    ptx::griddep_launch();
    const int64_t n = int64_t(B) * H * W * C;
    for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < n; i += int64_t(gridDim.x) * blockDim.x) {
        const int c = int(i % C);
        const int64_t p = i / C;
        const int w = int(p % W), h = int((p / W) % H), b = int(p / (int64_t(W) * H));
        float acc = 0.f;
        for (int r = 0; r < 3; ++r) {
            const int hh = h + 1 - r;
            if (hh < 0 || (hh & 1)) continue;
            const int ho = hh >> 1;
            if (ho >= Ho) continue;
            for (int s = 0; s < 3; ++s) {
                const int ww = w + 1 - s;
                if (ww < 0 || (ww & 1)) continue;
                const int wo = ww >> 1;
                if (wo >= Wo) continue;
                const size_t o = ((size_t(b) * Ho + ho) * Wo + wo) * C + c;
                if (arg[o] == r * 3 + s) acc += gout[o];
            }
        }
        gin[i] = acc;
    }
}

// Global average pool: act [B*HW][ld] -> pooled [B][C+1] (ones column at C for the fc bias).
template <int KIND>
__global__ void avgpool_kernel(CTensor act, int B, int HW, int C, CTensor pooled) {
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

// d act[b, k, c] = dpooled[b][c] / HW, fp32, 4 channels per thread.
__global__ void avgpool_backward_kernel(const float *dp, int ldp, int B, int HW, int C, float *g) {
    ptx::griddep_wait();
    ptx::griddep_launch();
    const int C4 = C / 4;
    const int64_t n = int64_t(B) * HW * C4;
    const float inv = 1.f / float(HW);
    for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < n; i += int64_t(gridDim.x) * blockDim.x) {
        const int c = int(i % C4) * 4;
        const int64_t r = i / C4;
        const float *s = dp + (r / HW) * ldp + c;
        st_f4(g, size_t(r) * C + c, make_float4(s[0] * inv, s[1] * inv, s[2] * inv, s[3] * inv));
    }
}

// Softmax cross-entropy for many classes (ImageNet heads): one CTA per sample,
// fixed-tree block reductions; per-sample losses summed in ascending sample
// order by loss_sum_kernel (ref _kernels.pyx:80-100 semantics).
template <int KIND>
__global__ void __launch_bounds__(256) xent_rows_kernel(const float *__restrict__ z, int B, int C, const int *perm,
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
        if (o == lab) loss_rows[s] = -log(double(pz));
    }
}

__global__ void loss_sum_kernel(const double *rows, int B, double *loss_out, unsigned *loss_flag) {
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

// The pre-hop waits of a weight hop (EpiWgrad::pre) in a one-CTA kernel ahead
// of the GEMM, so that a GEMM grid never occupies SMs while it waits for a peer
// (no dependent launch is triggered before the waits are over).
__global__ void hop_wait_kernel(HopParams p) { EpiWgrad<0>::pre(p, threadIdx.x, true); }

// Hop / update of a small parameter vector (batch-norm gamma|beta, gradient
// g[0..n) = [dgamma | dbeta] in the parameter order) with the same modes and
// ring protocol as the weight-gradient epilogue.  One CTA of 128 threads.
__global__ void vector_hop_kernel(HopParams p, const float *dgamma, const float *dbeta, int C) {
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
