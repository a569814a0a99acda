// Convolutional-network layer kernels for the ResNet configs (BASELINE
// configs[1..2,4]): convolutions run as tcgen05 GEMMs over an im2col matrix
// (NHWC activations, rows = output pixels, columns = (r, s, c) with c
// fastest), batch norm in training mode (per-micro-batch statistics, fp64
// reductions in a fixed order), residual adds, ReLU, global average pooling,
// and the vector hop / update for the batch-norm affine parameters.
//
// Activations are stored in the GEMM compute format (bf16, or fp32 hi/lo for
// the 3xTF32 mode); convolution outputs and all gradients flowing between
// layers are fp32.
#pragma once
#include "mlp_kernels.cuh"

namespace cdp {

// ---------------------------------------------------------------------------
// im2col: x NHWC [B*H*W][ld_x] (C channels) -> cols [B*Ho*Wo][ld_c], K = R*S*C
// columns (zero padding at borders, zero columns K..ld_c-1 for the TMA pad).
template <int KIND>
__global__ void im2col_kernel(CTensor x, int B, int H, int W, int C, int R, int S, int stride, int pad, int Ho,
                              int Wo, CTensor cols) {
    ptx::griddep_wait();
    ptx::griddep_launch();
    const int K = R * S * C;
    const int64_t rows = int64_t(B) * Ho * Wo;
    for (int64_t p = blockIdx.x; p < rows; p += gridDim.x) {
        const int wo = int(p % Wo), ho = int((p / Wo) % Ho), b = int(p / (int64_t(Wo) * Ho));
        for (int k = threadIdx.x; k < cols.ld; k += blockDim.x) {
            float v = 0.f;
            if (k < K) {
                const int c = k % C, rs = k / C, s = rs % S, r = rs / S;
                const int h = ho * stride - pad + r, w = wo * stride - pad + s;
                if (h >= 0 && h < H && w >= 0 && w < W)
                    v = Fmt<KIND>::load(x.hi, x.lo, (size_t(b) * H * W + size_t(h) * W + w) * x.ld + c);
            }
            Fmt<KIND>::store(cols.hi, cols.lo, size_t(p) * cols.ld + k, v);
        }
    }
}

// col2im (deterministic gather): dx[b,h,w,c] = sum over (r, s) ascending of
// dcols[(b, ho, wo), (r, s, c)] with h = ho*stride - pad + r.
__global__ void col2im_kernel(const float *__restrict__ dcols, int ldc, int B, int H, int W, int C, int R, int S,
                              int stride, int pad, int Ho, int Wo, float *dx, int ldx) {
    ptx::griddep_wait();
    ptx::griddep_launch();
    const int64_t n = int64_t(B) * H * W * C;
    for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < n; i += int64_t(gridDim.x) * blockDim.x) {
        const int c = int(i % C);
        const int64_t pix = i / C;
        const int w = int(pix % W), h = int((pix / W) % H), b = int(pix / (int64_t(W) * H));
        float acc = 0.f;
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
                acc += dcols[(size_t(b) * Ho * Wo + size_t(ho) * Wo + wo) * ldc + (r * S + s) * C + c];
            }
        }
        dx[size_t(pix) * ldx + c] = acc;
    }
}

// ---------------------------------------------------------------------------
// GEMM epilogue: fp32 row-major store (rows = pixels); used for convolution
// outputs (pre-BN) and im2col-space data gradients.
struct EpiRowF32 {
    struct Params {
        float *out;
        int ld;
    };
    struct State {};
    __device__ static void begin(const Params &, int, State &) {}
    __device__ static void apply(const Params &p, int m, int n0, const float (&v)[32], int M, int N, State &) {
        if (m >= M) return;
        float *row = p.out + size_t(m) * p.ld + n0;
        if (n0 + 32 <= N && ((p.ld | n0) & 3) == 0) {
#pragma unroll
            for (int i = 0; i < 32; i += 4) *reinterpret_cast<float4 *>(row + i) = make_float4(v[i], v[i + 1], v[i + 2], v[i + 3]);
        } else {
#pragma unroll
            for (int i = 0; i < 32; ++i)
                if (n0 + i < N) row[i] = v[i];
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
// Batch norm (training mode, ref: per micro-batch statistics).
// Column sums over rows of a [P][C] fp32 matrix, two deterministic passes:
// partial[blk][c] over a fixed row range, then the partials in block order.
// Computes sum(x) and sum(x^2) (forward) or sum(g) and sum(g * xhat) (backward).
constexpr int kBnRowsPerBlock = 256;

// mode 0: (x, x^2); mode 1: (g', g' * xhat) with g' = g masked by (a > 0) when mask != null
template <int KIND>
__global__ void bn_partial_kernel(const float *__restrict__ x, int ldx, int64_t P, int C, int mode,
                                  const float *__restrict__ g, int ldg, CTensor mask, const float *mean,
                                  const float *rstd, double *partial) {
    ptx::griddep_wait();
    ptx::griddep_launch();
    const int64_t r0 = int64_t(blockIdx.x) * kBnRowsPerBlock, r1 = min(P, r0 + kBnRowsPerBlock);
    for (int c = threadIdx.x; c < C; c += blockDim.x) {
        double s0 = 0.0, s1 = 0.0;
        if (mode == 0) {
            for (int64_t r = r0; r < r1; ++r) {
                const double v = x[r * ldx + c];
                s0 += v;
                s1 += v * v;
            }
        } else {
            const float mu = mean[c], rs = rstd[c];
            for (int64_t r = r0; r < r1; ++r) {
                float gv = g[r * ldg + c];
                if (mask.hi && !(Fmt<KIND>::load(mask.hi, mask.lo, size_t(r) * mask.ld + c) > 0.f)) gv = 0.f;
                const float xh = (x[r * ldx + c] - mu) * rs;
                s0 += gv;
                s1 += double(gv) * xh;
            }
        }
        partial[(size_t(blockIdx.x) * C + c) * 2] = s0;
        partial[(size_t(blockIdx.x) * C + c) * 2 + 1] = s1;
    }
}

// Forward finalise: mean, rstd (biased variance, eps) per channel.
// Backward finalise: out[0][c] = sum g' (dbeta), out[1][c] = sum g' xhat (dgamma).
__global__ void bn_finalize_kernel(const double *partial, int nblk, int C, int64_t P, int mode, float eps, float *a,
                                   float *b) {
    ptx::griddep_wait();
    ptx::griddep_launch();
    for (int c = blockIdx.x * blockDim.x + threadIdx.x; c < C; c += gridDim.x * blockDim.x) {
        double s0 = 0.0, s1 = 0.0;
        for (int k = 0; k < nblk; ++k) {
            s0 += partial[(size_t(k) * C + c) * 2];
            s1 += partial[(size_t(k) * C + c) * 2 + 1];
        }
        if (mode == 0) {
            const double mu = s0 / double(P);
            const double var = fmax(s1 / double(P) - mu * mu, 0.0);
            a[c] = float(mu);
            b[c] = float(1.0 / sqrt(var + double(eps)));
        } else {
            a[c] = float(s0);  // dbeta
            b[c] = float(s1);  // dgamma
        }
    }
}

// y = relu?( gamma * (x - mean) * rstd + beta  [+ residual] ) -> compute format.
// residual: either a compute-format tensor (identity shortcut) or a second
// BN-normalised fp32 tensor (projection shortcut).
struct BnResidual {
    CTensor act;           // identity shortcut (act.hi != null)
    const float *x;        // projection: conv output, its stats and affine
    int ldx;
    const float *mean, *rstd, *gamma, *beta;
};

template <int KIND>
__global__ void bn_apply_kernel(const float *__restrict__ x, int ldx, int64_t P, int C, const float *mean,
                                const float *rstd, const float *gamma, const float *beta, BnResidual res, int relu,
                                CTensor out) {
    ptx::griddep_wait();
    ptx::griddep_launch();
    const int64_t n = P * C;
    for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < n; i += int64_t(gridDim.x) * blockDim.x) {
        const int c = int(i % C);
        const int64_t r = i / C;
        float v = gamma[c] * ((x[r * ldx + c] - mean[c]) * rstd[c]) + beta[c];
        if (res.act.hi) v += Fmt<KIND>::load(res.act.hi, res.act.lo, size_t(r) * res.act.ld + c);
        if (res.x) v += res.gamma[c] * ((res.x[r * res.ldx + c] - res.mean[c]) * res.rstd[c]) + res.beta[c];
        if (relu) v = fmaxf(v, 0.f);
        Fmt<KIND>::store(out.hi, out.lo, size_t(r) * out.ld + c, v);
    }
}

// Backward through BN (+ReLU mask): dx = gamma * rstd * (g' - dbeta/P - xhat * dgamma/P)
// written in compute format (the conv's output gradient, a GEMM operand).
template <int KIND>
__global__ void bn_backward_kernel(const float *__restrict__ x, int ldx, int64_t P, int C, const float *mean,
                                   const float *rstd, const float *gamma, const float *dbeta, const float *dgamma,
                                   const float *__restrict__ g, int ldg, CTensor mask, CTensor dx) {
    ptx::griddep_wait();
    ptx::griddep_launch();
    const int64_t n = P * C;
    const float inv = 1.f / float(P);
    for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < n; i += int64_t(gridDim.x) * blockDim.x) {
        const int c = int(i % C);
        const int64_t r = i / C;
        float gv = g[r * ldg + c];
        if (mask.hi && !(Fmt<KIND>::load(mask.hi, mask.lo, size_t(r) * mask.ld + c) > 0.f)) gv = 0.f;
        const float xh = (x[r * ldx + c] - mean[c]) * rstd[c];
        const float d = gamma[c] * rstd[c] * (gv - dbeta[c] * inv - xh * dgamma[c] * inv);
        Fmt<KIND>::store(dx.hi, dx.lo, size_t(r) * dx.ld + c, d);
    }
}

// g_out = a + b (both fp32 [P][C]), optionally masking b by (act > 0) first.
template <int KIND>
__global__ void add_kernel(const float *a, const float *b, int ld, int64_t P, int C, CTensor mask_b, float *out) {
    ptx::griddep_wait();
    ptx::griddep_launch();
    const int64_t n = P * C;
    for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < n; i += int64_t(gridDim.x) * blockDim.x) {
        const int c = int(i % C);
        const int64_t r = i / C;
        float vb = b[r * ld + c];
        if (mask_b.hi && !(Fmt<KIND>::load(mask_b.hi, mask_b.lo, size_t(r) * mask_b.ld + c) > 0.f)) vb = 0.f;
        out[r * ld + c] = a[r * ld + c] + vb;
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

// d act[b, k, c] = dpooled[b][c] / HW, fp32.
__global__ void avgpool_backward_kernel(const float *dp, int ldp, int B, int HW, int C, float *g, int ldg) {
    ptx::griddep_wait();
    ptx::griddep_launch();
    const int64_t n = int64_t(B) * HW * C;
    for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < n; i += int64_t(gridDim.x) * blockDim.x) {
        const int c = int(i % C);
        const int64_t r = i / C;
        g[r * ldg + c] = dp[(r / HW) * ldp + c] / float(HW);
    }
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
