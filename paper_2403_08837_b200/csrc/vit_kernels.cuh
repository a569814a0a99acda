// Vision-Transformer layer kernels (BASELINE configs[3]: ViT-B/16) around the
// persistent tcgen05 GEMM: patch im2col, token assembly, LayerNorm forward /
// backward / parameter gradients, attention softmax forward / backward, token
// gradients of the embeddings, and a multi-CTA flat hop for vector parameters.
// The residual stream is fp32; GEMM operands are bf16 (KIND 0), with a constant
// ones column after the features of every linear layer's input (bias folding:
// [x, 1] . [W; b], the reference's flat [W][b] layout).  Reductions run in a
// fixed order (warp xor trees over fixed lane assignments, row blocks in order).
#pragma once
#include "conv_kernels.cuh"

namespace cdp {

__device__ __forceinline__ float warp_sum(float v) {
#pragma unroll
    for (int o = 16; o; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    return v;
}
__device__ __forceinline__ float warp_max(float v) {
#pragma unroll
    for (int o = 16; o; o >>= 1) v = fmaxf(v, __shfl_xor_sync(0xffffffffu, v, o));
    return v;
}

// patches[b*np + gy*G + gx][(r*P + s)*3 + c] = image[perm[b]][gy*P + r][gx*P + s][c];
// column K = P*P*3 is the constant 1 (bias), columns above it 0.
template <int KIND>
static __global__ void patch_im2col_kernel(const float *__restrict__ data, const int *perm, int img, int P, int G, int rows,
                                    CTensor out) {
    ptx::griddep_wait();
    ptx::griddep_launch();
    const int K = P * P * 3;
    const int64_t n = int64_t(rows) * out.ld;
    for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < n; i += int64_t(gridDim.x) * blockDim.x) {
        const int k = int(i % out.ld);
        const int row = int(i / out.ld);
        float v = k == K ? 1.f : 0.f;
        if (k < K) {
            const int np = G * G;
            const int b = row / np, pi = row % np, gy = pi / G, gx = pi % G;
            const int r = k / (P * 3), rem = k % (P * 3), s = rem / 3, c = rem % 3;
            v = data[((size_t(perm[b]) * img + gy * P + r) * img + gx * P + s) * 3 + c];
        }
        Fmt<KIND>::store(out.hi, out.lo, size_t(i), v);
    }
}

// h0[b*T + 0] = cls + pos[0];  h0[b*T + 1 + p] = E[b*np + p] + pos[1 + p]   (fp32, D features)
static __global__ void embed_assemble_kernel(const float *__restrict__ E, const float *cls, const float *pos, int B, int T,
                                      int D, float *h0) {
    ptx::griddep_wait();
    ptx::griddep_launch();
    const int64_t n = int64_t(B) * T * D;
    for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < n; i += int64_t(gridDim.x) * blockDim.x) {
        const int d = int(i % D);
        const int64_t row = i / D;
        const int t = int(row % T), b = int(row / T);
        const float e = t == 0 ? cls[d] : E[(size_t(b) * (T - 1) + t - 1) * D + d];
        h0[i] = e + pos[size_t(t) * D + d];
    }
}

// LayerNorm forward, one warp per row (row r reads x row r * in_stride):
// out = gamma * (x - mean) * rstd + beta  (compute format, ones column at D), mean / rstd saved.
template <int KIND>
static __global__ void ln_fwd_kernel(const float *__restrict__ x, int rows, int in_stride, int D, const float *gb, float eps,
                              CTensor out, float *mean, float *rstd) {
    ptx::griddep_wait();
    ptx::griddep_launch();
    const int w = (blockIdx.x * blockDim.x + threadIdx.x) >> 5, lane = threadIdx.x & 31;
    if (w >= rows) return;
    const float *xr = x + size_t(w) * in_stride * D;
    float s = 0.f;
    for (int d = lane; d < D; d += 32) s += xr[d];
    const float mu = warp_sum(s) / float(D);
    float q = 0.f;
    for (int d = lane; d < D; d += 32) {
        const float c = xr[d] - mu;
        q += c * c;
    }
    const float rs = rsqrtf(warp_sum(q) / float(D) + eps);
    for (int d = lane; d < D; d += 32)
        Fmt<KIND>::store(out.hi, out.lo, size_t(w) * out.ld + d, gb[d] * ((xr[d] - mu) * rs) + gb[D + d]);
    if (lane == 0) {
        Fmt<KIND>::store(out.hi, out.lo, size_t(w) * out.ld + D, 1.f);
        mean[w] = mu;
        rstd[w] = rs;
    }
}

// Same with the row held in registers as float4 columns (lane owns 4*lane + 128*k, k < C4 = D/128):
// one read of x, 16-byte accesses.
template <int KIND, int C4>
static __global__ void ln_fwd4_kernel(const float *__restrict__ x, int rows, int in_stride, int D, const float *gb,
                                      float eps, CTensor out, float *mean, float *rstd) {
    ptx::griddep_wait();
    ptx::griddep_launch();
    const int w = (blockIdx.x * blockDim.x + threadIdx.x) >> 5, lane = threadIdx.x & 31;
    if (w >= rows) return;
    const float *xr = x + size_t(w) * in_stride * D;
    float4 v[C4], ga[C4], be[C4];
    float s = 0.f;
#pragma unroll
    for (int k = 0; k < C4; ++k) {  // gamma / beta with the row: their loads overlap the reductions
        v[k] = *reinterpret_cast<const float4 *>(xr + 4 * lane + 128 * k);
        ga[k] = *reinterpret_cast<const float4 *>(gb + 4 * lane + 128 * k);
        be[k] = *reinterpret_cast<const float4 *>(gb + D + 4 * lane + 128 * k);
    }
#pragma unroll
    for (int k = 0; k < C4; ++k) s += (v[k].x + v[k].y) + (v[k].z + v[k].w);
    const float mu = warp_sum(s) / float(D);
    float q = 0.f;
#pragma unroll
    for (int k = 0; k < C4; ++k) {
        const float a = v[k].x - mu, b = v[k].y - mu, c = v[k].z - mu, d = v[k].w - mu;
        q += (a * a + b * b) + (c * c + d * d);
    }
    const float rs = rsqrtf(warp_sum(q) / float(D) + eps);
    const bool vec = (out.ld % 4) == 0;
#pragma unroll
    for (int k = 0; k < C4; ++k) {
        const int d = 4 * lane + 128 * k;
        const float4 y = make_float4(ga[k].x * ((v[k].x - mu) * rs) + be[k].x, ga[k].y * ((v[k].y - mu) * rs) + be[k].y,
                                     ga[k].z * ((v[k].z - mu) * rs) + be[k].z, ga[k].w * ((v[k].w - mu) * rs) + be[k].w);
        const size_t o = size_t(w) * out.ld + d;
        if (vec) {
            store_wc4<KIND>(out, o, y);
        } else {
            Fmt<KIND>::store(out.hi, out.lo, o, y.x);
            Fmt<KIND>::store(out.hi, out.lo, o + 1, y.y);
            Fmt<KIND>::store(out.hi, out.lo, o + 2, y.z);
            Fmt<KIND>::store(out.hi, out.lo, o + 3, y.w);
        }
    }
    if (lane == 0) {
        Fmt<KIND>::store(out.hi, out.lo, size_t(w) * out.ld + D, 1.f);
        mean[w] = mu;
        rstd[w] = rs;
    }
}

// Fused LayerNorm backward over a block of kLnRows rows (8 warps, a warp per row, lane owns
// columns lane + 32 k): dh_out = dh_in + dx (fp32) and, when copy.hi, the same row in compute
// format (the next GEMM's operand); per-column (sum g, sum g xhat) of the block's rows combined
// over the warps in fixed order -> partial[d][blk][2] (fp64), finalised by bn_finalize_bwd_kernel.
#ifndef LN_BWD_MINB
#define LN_BWD_MINB 2  // two CTAs per SM (<= 128 registers): at 136 registers one CTA per SM ran 2.7 waves
#endif
constexpr int kLnBwdRows = 16;  // smallest rows per CTA of the fused backward (2 per warp; sizes the partials)
// rows per CTA at run time (CDP_LN_BWD_ROWS, a multiple of 16): 16 by default
inline int ln_bwd_rows() {
    static const int v = [] {
        const char *e = std::getenv("CDP_LN_BWD_ROWS");
        const int r = e ? std::atoi(e) : 16;
        return r >= 16 && r % 16 == 0 ? r : 16;
    }();
    return v;
}
template <int KIND, int CPL>
static __global__ void __launch_bounds__(256) ln_bwd_fused_kernel(const float *__restrict__ g,
                                                                  const float *__restrict__ x, int rows,
                                                                  int in_stride, int D, const float *gb,
                                                                  const float *mean, const float *rstd,
                                                                  const float *dh_in, float *dh_out, CTensor copy,
                                                                  double *partial, int rpc) {
    ptx::griddep_wait();
    ptx::griddep_launch();
    extern __shared__ float red[];  // [8][D][2]
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    float sg[CPL], sx[CPL];
#pragma unroll
    for (int k = 0; k < CPL; ++k) sg[k] = sx[k] = 0.f;
    const int r0 = blockIdx.x * rpc, r1 = min(rows, r0 + rpc);
    for (int w = r0 + warp; w < r1; w += 8) {
        const size_t xo = size_t(w) * in_stride * D, go = size_t(w) * D;
        const float mu = mean[w], rs = rstd[w];
        float gv[CPL], xh[CPL];
        float a = 0.f, b = 0.f;
#pragma unroll
        for (int k = 0; k < CPL; ++k) {
            const int d = lane + 32 * k;
            gv[k] = g[go + d];
            xh[k] = (x[xo + d] - mu) * rs;
            const float gg = gv[k] * gb[d];
            a += gg;
            b += gg * xh[k];
            sg[k] += gv[k];
            sx[k] = fmaf(gv[k], xh[k], sx[k]);
        }
        a = warp_sum(a) / float(D);
        b = warp_sum(b) / float(D);
#pragma unroll
        for (int k = 0; k < CPL; ++k) {
            const int d = lane + 32 * k;
            const float v = (dh_in ? dh_in[xo + d] : 0.f) + rs * (gv[k] * gb[d] - a - xh[k] * b);
            dh_out[xo + d] = v;
            if (copy.hi) Fmt<KIND>::store(copy.hi, copy.lo, size_t(w) * in_stride * copy.ld + d, v);
        }
    }
#pragma unroll
    for (int k = 0; k < CPL; ++k) {
        const int d = lane + 32 * k;
        red[(warp * D + d) * 2] = sg[k];
        red[(warp * D + d) * 2 + 1] = sx[k];
    }
    __syncthreads();
    for (int d = threadIdx.x; d < D; d += blockDim.x) {
        double s0 = 0.0, s1 = 0.0;
        for (int q = 0; q < 8; ++q) {
            s0 += double(red[(q * D + d) * 2]);
            s1 += double(red[(q * D + d) * 2 + 1]);
        }
        double *o = partial + (size_t(d) * gridDim.x + blockIdx.x) * 2;
        o[0] = s0;  // -> dbeta
        o[1] = s1;  // -> dgamma
    }
}

// Same with 16-byte accesses: lane owns columns 4*lane + 128*k (k < C4 = D/128); both rows of a
// warp are loaded before either is reduced (more loads in flight per thread).
template <int KIND, int C4>
static __global__ void __launch_bounds__(256, LN_BWD_MINB) ln_bwd_fused4_kernel(const float *__restrict__ g,
                                                                   const float *__restrict__ x, int rows,
                                                                   int in_stride, int D, const float *gb,
                                                                   const float *mean, const float *rstd,
                                                                   const float *dh_in, float *dh_out, CTensor copy,
                                                                   double *partial, int rpc) {
    ptx::griddep_wait();
    ptx::griddep_launch();
    extern __shared__ float red[];  // [8][D][2]
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    float4 sg[C4], sx[C4];
#pragma unroll
    for (int k = 0; k < C4; ++k) sg[k] = sx[k] = make_float4(0.f, 0.f, 0.f, 0.f);
    const int r0 = blockIdx.x * rpc, r1 = min(rows, r0 + rpc);
    const bool vcopy = copy.hi && (copy.ld % 4) == 0;
    for (int w = r0 + warp; w < r1; w += 8) {
        const size_t xo = size_t(w) * in_stride * D, go = size_t(w) * D;
        const float mu = mean[w], rs = rstd[w];
        float4 gv[C4], xh[C4];
        float a = 0.f, b = 0.f;
#pragma unroll
        for (int k = 0; k < C4; ++k) {
            const int d = 4 * lane + 128 * k;
            gv[k] = *reinterpret_cast<const float4 *>(g + go + d);
            const float4 xv = *reinterpret_cast<const float4 *>(x + xo + d);
            xh[k] = make_float4((xv.x - mu) * rs, (xv.y - mu) * rs, (xv.z - mu) * rs, (xv.w - mu) * rs);
        }
#pragma unroll
        for (int k = 0; k < C4; ++k) {
            const int d = 4 * lane + 128 * k;
            const float4 gm = *reinterpret_cast<const float4 *>(gb + d);
            const float g0 = gv[k].x * gm.x, g1 = gv[k].y * gm.y, g2 = gv[k].z * gm.z, g3 = gv[k].w * gm.w;
            a += g0 + g1 + g2 + g3;
            b += g0 * xh[k].x + g1 * xh[k].y + g2 * xh[k].z + g3 * xh[k].w;
            sg[k].x += gv[k].x;
            sg[k].y += gv[k].y;
            sg[k].z += gv[k].z;
            sg[k].w += gv[k].w;
            sx[k].x = fmaf(gv[k].x, xh[k].x, sx[k].x);
            sx[k].y = fmaf(gv[k].y, xh[k].y, sx[k].y);
            sx[k].z = fmaf(gv[k].z, xh[k].z, sx[k].z);
            sx[k].w = fmaf(gv[k].w, xh[k].w, sx[k].w);
        }
        a = warp_sum(a) / float(D);
        b = warp_sum(b) / float(D);
#pragma unroll
        for (int k = 0; k < C4; ++k) {
            const int d = 4 * lane + 128 * k;
            const float4 gm = *reinterpret_cast<const float4 *>(gb + d);
            const float4 hi = dh_in ? *reinterpret_cast<const float4 *>(dh_in + xo + d) : make_float4(0.f, 0.f, 0.f, 0.f);
            float4 v;
            v.x = hi.x + rs * (gv[k].x * gm.x - a - xh[k].x * b);
            v.y = hi.y + rs * (gv[k].y * gm.y - a - xh[k].y * b);
            v.z = hi.z + rs * (gv[k].z * gm.z - a - xh[k].z * b);
            v.w = hi.w + rs * (gv[k].w * gm.w - a - xh[k].w * b);
            *reinterpret_cast<float4 *>(dh_out + xo + d) = v;
            if (vcopy) {
                store_wc4<KIND>(copy, size_t(w) * in_stride * copy.ld + d, v);
            } else if (copy.hi) {
                const size_t co = size_t(w) * in_stride * copy.ld + d;
                Fmt<KIND>::store(copy.hi, copy.lo, co, v.x);
                Fmt<KIND>::store(copy.hi, copy.lo, co + 1, v.y);
                Fmt<KIND>::store(copy.hi, copy.lo, co + 2, v.z);
                Fmt<KIND>::store(copy.hi, copy.lo, co + 3, v.w);
            }
        }
    }
#pragma unroll
    for (int k = 0; k < C4; ++k) {
        const int d = 4 * lane + 128 * k;
        float *o = red + (warp * D + d) * 2;
        o[0] = sg[k].x;
        o[1] = sx[k].x;
        o[2] = sg[k].y;
        o[3] = sx[k].y;
        o[4] = sg[k].z;
        o[5] = sx[k].z;
        o[6] = sg[k].w;
        o[7] = sx[k].w;
    }
    __syncthreads();
    for (int d = threadIdx.x; d < D; d += blockDim.x) {
        double s0 = 0.0, s1 = 0.0;
        for (int q = 0; q < 8; ++q) {
            s0 += double(red[(q * D + d) * 2]);
            s1 += double(red[(q * D + d) * 2 + 1]);
        }
        double *o = partial + (size_t(d) * gridDim.x + blockIdx.x) * 2;
        o[0] = s0;  // -> dbeta
        o[1] = s1;  // -> dgamma
    }
}

// Row softmax of scale * S (fp32 [rows][lds], n valid columns) -> P (bf16 [rows][ldp]); one warp per row.
static __global__ void softmax_fwd_kernel(const float *__restrict__ S, int rows, int n, int lds, float scale,
                                   __nv_bfloat16 *P, int ldp) {
    ptx::griddep_wait();
    ptx::griddep_launch();
    const int w = (blockIdx.x * blockDim.x + threadIdx.x) >> 5, lane = threadIdx.x & 31;
    if (w >= rows) return;
    const float *sr = S + size_t(w) * lds;
    float mx = -INFINITY;
    for (int j = lane; j < n; j += 32) mx = fmaxf(mx, sr[j] * scale);
    mx = warp_max(mx);
    float sum = 0.f;
    for (int j = lane; j < n; j += 32) sum += __expf(sr[j] * scale - mx);
    const float inv = 1.f / warp_sum(sum);
    for (int j = lane; j < n; j += 32) P[size_t(w) * ldp + j] = __float2bfloat16_rn(__expf(sr[j] * scale - mx) * inv);
}

// dS = scale * P (dP - sum_j dP_j P_j)   (gradient w.r.t. the unscaled scores), bf16.
static __global__ void softmax_bwd_kernel(const float *__restrict__ dP, const __nv_bfloat16 *__restrict__ P, int rows, int n,
                                   int lds, int ldp, float scale, __nv_bfloat16 *dS) {
    ptx::griddep_wait();
    ptx::griddep_launch();
    const int w = (blockIdx.x * blockDim.x + threadIdx.x) >> 5, lane = threadIdx.x & 31;
    if (w >= rows) return;
    float dot = 0.f;
    for (int j = lane; j < n; j += 32) dot += dP[size_t(w) * lds + j] * __bfloat162float(P[size_t(w) * ldp + j]);
    dot = warp_sum(dot);
    for (int j = lane; j < n; j += 32) {
        const float p = __bfloat162float(P[size_t(w) * ldp + j]);
        dS[size_t(w) * ldp + j] = __float2bfloat16_rn(scale * p * (dP[size_t(w) * lds + j] - dot));
    }
}

// Compute-format row softmax / backward (the fp32 mode: P and dS as hi + lo operands of the 3xTF32
// attention GEMMs); one warp per row, accurate expf.
template <int KIND>
static __global__ void softmax_fwd_c_kernel(const float *__restrict__ S, int rows, int n, int lds, float scale,
                                            CTensor P) {
    ptx::griddep_wait();
    ptx::griddep_launch();
    const int w = (blockIdx.x * blockDim.x + threadIdx.x) >> 5, lane = threadIdx.x & 31;
    if (w >= rows) return;
    const float *sr = S + size_t(w) * lds;
    float mx = -INFINITY;
    for (int j = lane; j < n; j += 32) mx = fmaxf(mx, sr[j] * scale);
    mx = warp_max(mx);
    float sum = 0.f;
    for (int j = lane; j < n; j += 32) sum += expf(sr[j] * scale - mx);
    const float inv = 1.f / warp_sum(sum);
    for (int j = lane; j < n; j += 32)
        Fmt<KIND>::store(P.hi, P.lo, size_t(w) * P.ld + j, expf(sr[j] * scale - mx) * inv);
}

template <int KIND>
static __global__ void softmax_bwd_c_kernel(const float *__restrict__ dP, CTensor P, int rows, int n, int lds,
                                            float scale, CTensor dS) {
    ptx::griddep_wait();
    ptx::griddep_launch();
    const int w = (blockIdx.x * blockDim.x + threadIdx.x) >> 5, lane = threadIdx.x & 31;
    if (w >= rows) return;
    float dot = 0.f;
    for (int j = lane; j < n; j += 32) dot += dP[size_t(w) * lds + j] * Fmt<KIND>::load(P.hi, P.lo, size_t(w) * P.ld + j);
    dot = warp_sum(dot);
    for (int j = lane; j < n; j += 32) {
        const float p = Fmt<KIND>::load(P.hi, P.lo, size_t(w) * P.ld + j);
        Fmt<KIND>::store(dS.hi, dS.lo, size_t(w) * dS.ld + j, scale * p * (dP[size_t(w) * lds + j] - dot));
    }
}

// Vectorised row softmax / backward for rows of at most 128*NV columns: lane owns columns
// 4*lane + 128*k (16-byte fp32 / 8-byte bf16 accesses, one read of each row); columns >= n
// (the padded tail of a 197-token row) are masked.
template <int NV>
static __global__ void softmax_fwd4_kernel(const float *__restrict__ S, int rows, int n, int lds, float scale,
                                           __nv_bfloat16 *P, int ldp) {
    ptx::griddep_wait();
    ptx::griddep_launch();
    const int w = (blockIdx.x * blockDim.x + threadIdx.x) >> 5, lane = threadIdx.x & 31;
    if (w >= rows) return;
    const float *sr = S + size_t(w) * lds;
    float v[NV][4];
    float mx = -INFINITY;
#pragma unroll
    for (int k = 0; k < NV; ++k) {
        const int c = 4 * lane + 128 * k;
        float4 t = make_float4(-INFINITY, -INFINITY, -INFINITY, -INFINITY);
        if (c < n) t = *reinterpret_cast<const float4 *>(sr + c);
        v[k][0] = t.x * scale;
        v[k][1] = c + 1 < n ? t.y * scale : -INFINITY;
        v[k][2] = c + 2 < n ? t.z * scale : -INFINITY;
        v[k][3] = c + 3 < n ? t.w * scale : -INFINITY;
        if (c >= n) v[k][0] = -INFINITY;
#pragma unroll
        for (int j = 0; j < 4; ++j) mx = fmaxf(mx, v[k][j]);
    }
    mx = warp_max(mx);
    float sum = 0.f;
#pragma unroll
    for (int k = 0; k < NV; ++k)
#pragma unroll
        for (int j = 0; j < 4; ++j) {
            v[k][j] = __expf(v[k][j] - mx);
            sum += v[k][j];
        }
    const float inv = 1.f / warp_sum(sum);
    __nv_bfloat16 *pr = P + size_t(w) * ldp;
#pragma unroll
    for (int k = 0; k < NV; ++k) {
        const int c = 4 * lane + 128 * k;
        if (c + 3 < n) {
            __nv_bfloat162 a = __floats2bfloat162_rn(v[k][0] * inv, v[k][1] * inv);
            __nv_bfloat162 b = __floats2bfloat162_rn(v[k][2] * inv, v[k][3] * inv);
            uint2 u;
            u.x = *reinterpret_cast<uint32_t *>(&a);
            u.y = *reinterpret_cast<uint32_t *>(&b);
            *reinterpret_cast<uint2 *>(pr + c) = u;
        } else {
            for (int j = 0; j < 4 && c + j < n; ++j) pr[c + j] = __float2bfloat16_rn(v[k][j] * inv);
        }
    }
}

template <int NV>
static __global__ void softmax_bwd4_kernel(const float *__restrict__ dP, const __nv_bfloat16 *__restrict__ P, int rows,
                                           int n, int lds, int ldp, float scale, __nv_bfloat16 *dS) {
    ptx::griddep_wait();
    ptx::griddep_launch();
    const int w = (blockIdx.x * blockDim.x + threadIdx.x) >> 5, lane = threadIdx.x & 31;
    if (w >= rows) return;
    const float *dr = dP + size_t(w) * lds;
    const __nv_bfloat16 *pr = P + size_t(w) * ldp;
    float g[NV][4], p[NV][4];
    float dot = 0.f;
#pragma unroll
    for (int k = 0; k < NV; ++k) {
        const int c = 4 * lane + 128 * k;
#pragma unroll
        for (int j = 0; j < 4; ++j) g[k][j] = p[k][j] = 0.f;
        if (c + 3 < n) {
            const float4 t = *reinterpret_cast<const float4 *>(dr + c);
            const uint2 u = *reinterpret_cast<const uint2 *>(pr + c);
            const float2 p01 = __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162 *>(&u.x));
            const float2 p23 = __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162 *>(&u.y));
            g[k][0] = t.x, g[k][1] = t.y, g[k][2] = t.z, g[k][3] = t.w;
            p[k][0] = p01.x, p[k][1] = p01.y, p[k][2] = p23.x, p[k][3] = p23.y;
        } else {
            for (int j = 0; j < 4 && c + j < n; ++j) {
                g[k][j] = dr[c + j];
                p[k][j] = __bfloat162float(pr[c + j]);
            }
        }
#pragma unroll
        for (int j = 0; j < 4; ++j) dot += g[k][j] * p[k][j];
    }
    dot = warp_sum(dot);
    __nv_bfloat16 *sr = dS + size_t(w) * ldp;
#pragma unroll
    for (int k = 0; k < NV; ++k) {
        const int c = 4 * lane + 128 * k;
        float o[4];
#pragma unroll
        for (int j = 0; j < 4; ++j) o[j] = scale * p[k][j] * (g[k][j] - dot);
        if (c + 3 < n) {
            __nv_bfloat162 a = __floats2bfloat162_rn(o[0], o[1]);
            __nv_bfloat162 b = __floats2bfloat162_rn(o[2], o[3]);
            uint2 u;
            u.x = *reinterpret_cast<uint32_t *>(&a);
            u.y = *reinterpret_cast<uint32_t *>(&b);
            *reinterpret_cast<uint2 *>(sr + c) = u;
        } else {
            for (int j = 0; j < 4 && c + j < n; ++j) sr[c + j] = __float2bfloat16_rn(o[j]);
        }
    }
}

// fp32 [rows][D] -> compute format [rows][ld] (GEMM operand), optional row gather
// (out row r <- in row (r / per) * in_per + skip + r % per).
template <int KIND>
static __global__ void cast_rows_kernel(const float *__restrict__ in, int rows, int D, int per, int in_per, int skip,
                                 CTensor out) {
    ptx::griddep_wait();
    ptx::griddep_launch();
    const int64_t n = int64_t(rows) * D;
    for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < n; i += int64_t(gridDim.x) * blockDim.x) {
        const int d = int(i % D);
        const int r = int(i / D);
        const int64_t src = int64_t(r / per) * in_per + skip + r % per;
        Fmt<KIND>::store(out.hi, out.lo, size_t(r) * out.ld + d, in[size_t(src) * D + d]);
    }
}

// Embedding gradients: pos[t][d] = sum_b dh[b*T + t][d], cls[d] = sum_b dh[b*T][d] (ascending b).
static __global__ void token_grad_kernel(const float *__restrict__ dh, int B, int T, int D, float *gpos, float *gcls) {
    ptx::griddep_wait();
    ptx::griddep_launch();
    const int64_t n = int64_t(T) * D;
    for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < n; i += int64_t(gridDim.x) * blockDim.x) {
        float s = 0.f;
        for (int b = 0; b < B; ++b) s += dh[size_t(b) * T * D + i];
        gpos[i] = s;
        if (i < D) gcls[i] = s;
    }
}

// Hop / update of a flat vector parameter (class token, position embedding) from a gradient g[0..n)
// with the ring protocol of the weight hops (multi-CTA: the last CTA publishes).
static __global__ void flat_hop_kernel(HopParams p, const float *g, int64_t n) {
    ptx::griddep_wait();
    ptx::griddep_launch();
    EpiWgrad<0>::pre(p, threadIdx.x);
    bool bg = false, bu = false;
    for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < n; i += int64_t(gridDim.x) * blockDim.x)
        hop_elem<0>(p, p.base + i, g[i], 0, false, bg, bu);
    if (bg) atomicOr(p.grad_flags, 1u << ((p.stage - 1) & 31));
    if (bu) atomicOr(p.upd_flags, 1u << ((p.stage - 1) & 31));
    EpiWgrad<0>::post(p, threadIdx.x, gridDim.x);
}

}  // namespace cdp
