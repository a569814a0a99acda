// Fused multi-head attention for the ViT trainer (sm_100a, bf16 operands, fp32 TMEM accumulators).
//
// Forward: one CTA per (query tile, head, sample); backward: one per (head, sample).  The whole key range of a ViT-B/16 sequence (T = 197 <= 256) is one
// tile, so the softmax is exact in one pass over a 128 x 256 score tile held in TMEM — no online
// rescaling — and only the per-row log-sum-exp leaves the forward (the backward recomputes the
// probabilities from it, flash-attention style).  Replaces the batched score / value GEMMs, the
// fp32 score tensor and the row-softmax kernels of the unfused path (vit_trainer.cu), whose
// [B][H][T][T] score / probability tensors were 60-100 MB of HBM traffic per layer.
//
// Operands are 4-D TMA views {64 dims, T tokens, H heads, B samples} of the token-major qkv / dO
// buffers (rows beyond T are out-of-bounds zero fill).  Shared-memory tiles use the 128-byte swizzle;
// the same [rows][64] tile serves as a K-major operand (Q K^T) and as an MN-major one (P V, dS K,
// dS^T Q, P^T dO), and the probability / dS tile [128 queries][256 keys] (four 64-key chunks of
// [128 rows][128 B]) is a K-major A operand (P V, dS K) and, transposed, an MN-major one (P^T dO,
// dS^T Q).  Warp roles: 0 TMA, 1 MMA issue, 2 TMEM allocation, 4-7 softmax / epilogue (thread =
// tile row = TMEM lane).
#pragma once
#include <cuda_bf16.h>

#include "ptx.cuh"

namespace cdp {

struct AttnMaps {
    CUtensorMap q, k, v, dout;  // q / dout boxes {64, 128}, k / v boxes {64, 256}
};

struct AttnArgs {
    int T, H, B;
    float scale;                  // softmax scale (1 / sqrt(head dim))
    __nv_bfloat16 *o;             // O rows (b * T + t), columns h * 64 .. + 63 (forward output, backward input)
    int64_t o_ld;
    float *lse;                   // [(b * H + h) * T + t]: natural log-sum-exp of the scaled score row
    const __nv_bfloat16 *dout;    // backward: dO, same layout as O
    int64_t dout_ld;
    __nv_bfloat16 *dqkv;          // backward: dQ at column h * 64, dK at dk_off + h * 64, dV at dv_off + h * 64
    int64_t dqkv_ld, dk_off, dv_off;
};

constexpr int kAttnThreads = 256;
constexpr int kAttnFwdSmem = 98304 + 256 + 1024;
constexpr int kAttnBwdSmem = 163840 + 256 + 1024;
constexpr float kLog2e = 1.4426950408889634f;

namespace attn {
__device__ __forceinline__ uint64_t desc_k(uint32_t addr) { return ptx::smem_desc_sw128(addr, 16, 1024); }
// MN-major tile: 64-element chunks `lbo` bytes apart, 128-byte K rows
__device__ __forceinline__ uint64_t desc_mn(uint32_t addr, uint32_t lbo) { return ptx::smem_desc_sw128(addr, lbo, 1024); }
constexpr uint32_t kIdS = ptx::instr_desc(1, false, false, 128, 256);   // S = Q K^T, dP = dO V^T
constexpr uint32_t kIdO = ptx::instr_desc(1, false, true, 128, 64);     // O = P V, dQ = dS K
constexpr uint32_t kIdT = ptx::instr_desc(1, true, true, 128, 64);      // dV = P^T dO, dK = dS^T Q
// 16-byte unit u (8 keys) of row r in a 64-key chunk of the probability tile
__device__ __forceinline__ uint32_t p_off(int r, int key) {
    return uint32_t((key >> 6) * 16384 + r * 128 + ((((key & 63) >> 3) ^ (r & 7)) << 4));
}
__device__ __forceinline__ uint32_t pack2(float a, float b) {
    __nv_bfloat162 h = __floats2bfloat162_rn(a, b);
    return *reinterpret_cast<uint32_t *>(&h);
}
__device__ __forceinline__ float bf_lo(uint32_t u) { return __uint_as_float(u << 16); }
__device__ __forceinline__ float bf_hi(uint32_t u) { return __uint_as_float(u & 0xffff0000u); }
__device__ __forceinline__ uint8_t *align1024(uint8_t *p) {
    return p + ((1024u - (ptx::smem_u32(p) & 1023u)) & 1023u);
}
}  // namespace attn

// ---------------------------------------------------------------- forward
// One CTA per (query tile, head, sample).  Shared memory: [0, 64 KB) holds Q (16 KB) and K (32 KB) for
// the score MMA and then the probability tile (64 KB) over them; V at 64 KB: 96 KB and 256 TMEM
// columns, so two CTAs share an SM (one's softmax overlaps the other's loads and MMAs).
__global__ void __launch_bounds__(kAttnThreads, 2) attn_fwd_kernel(const __grid_constant__ AttnMaps maps, const AttnArgs a) {
    using namespace attn;
    extern __shared__ __align__(16) uint8_t smem_raw[];
    uint8_t *smem = align1024(smem_raw);
    uint8_t *sQ = smem, *sK = smem + 16384, *sP = smem, *sV = smem + 65536;
    uint64_t *bars = reinterpret_cast<uint64_t *>(smem + 98304);
    uint64_t *bar_in = bars, *bar_s = bars + 1, *bar_p = bars + 2, *bar_o = bars + 3;
    uint32_t *tmem_slot = reinterpret_cast<uint32_t *>(bars + 8);
    const int warp = int(ptx::warp_id()), lane = int(ptx::lane_id());
    const int T = a.T, ntile = (T + 127) / 128;
    const int i = int(blockIdx.x) % ntile, g = int(blockIdx.x) / ntile;
    const int h = g % a.H, b = g / a.H;
    if (warp == 0 && lane == 0) {
        ptx::tma_prefetch_desc(&maps.q);
        ptx::tma_prefetch_desc(&maps.k);
        ptx::tma_prefetch_desc(&maps.v);
    }
    if (warp == 1 && lane == 0) {
        ptx::mbar_init(bar_in, 1);
        ptx::mbar_init(bar_s, 1);
        ptx::mbar_init(bar_p, 4);
        ptx::mbar_init(bar_o, 1);
        ptx::fence_barrier_init();
    }
    if (warp == 2) ptx::tmem_alloc<256>(tmem_slot);
    ptx::tc_fence_before();
    __syncthreads();
    ptx::tc_fence_after();
    const uint32_t tmem = *tmem_slot;
    ptx::griddep_wait();
    ptx::griddep_launch();
    if (warp == 0) {
        if (lane == 0) {
            ptx::mbar_arrive_expect_tx(bar_in, 16384 + 65536);
            ptx::tma_load_4d(sQ, &maps.q, bar_in, 0, i * 128, h, b);
            ptx::tma_load_4d(sK, &maps.k, bar_in, 0, 0, h, b);
            ptx::tma_load_4d(sV, &maps.v, bar_in, 0, 0, h, b);
        }
    } else if (warp == 1) {
        if (lane == 0) {
            const uint32_t qa = ptx::smem_u32(sQ), ka = ptx::smem_u32(sK), va = ptx::smem_u32(sV),
                           pa = ptx::smem_u32(sP);
            const int ksteps = (T + 15) / 16;  // 16-key MMA steps of P V (the rest of P is zero)
            ptx::mbar_wait(bar_in, 0);
            ptx::tc_fence_after();
#pragma unroll
            for (int k = 0; k < 4; ++k) ptx::umma<0>(tmem, desc_k(qa + k * 32), desc_k(ka + k * 32), kIdS, k > 0);
            ptx::umma_commit(bar_s);  // (Q and K are free once it arrives: P is written over them)
            ptx::mbar_wait(bar_p, 0);
            ptx::tc_fence_after();
            for (int k = 0; k < ksteps; ++k)
                ptx::umma<0>(tmem, desc_k(pa + (k >> 2) * 16384 + (k & 3) * 32), desc_mn(va + k * 2048, 8192), kIdO,
                             k > 0);
            ptx::umma_commit(bar_o);
        }
    } else if (warp >= 4) {
        const int q = warp & 3, r = q * 32 + lane;
        const uint32_t trow = tmem + (uint32_t(q * 32) << 16);
        const float sl2 = a.scale * kLog2e;
        const int t = i * 128 + r;
        ptx::mbar_wait(bar_s, 0);
        ptx::tc_fence_after();
        float mx = -INFINITY;
#pragma unroll 1
        for (int c = 0; c * 32 < T; ++c) {
            float v[32];
            ptx::tmem_ld32(trow + c * 32, v);
#pragma unroll
            for (int j = 0; j < 32; ++j)
                if (c * 32 + j < T) mx = fmaxf(mx, v[j]);
        }
        const float off = mx * sl2;
        float sum = 0.f;
#pragma unroll 1
        for (int c = 0; c < 8; ++c) {  // every 32-key group of the tile (zeros past T)
            float v[32];
            if (c * 32 < T) ptx::tmem_ld32(trow + c * 32, v);
#pragma unroll
            for (int j = 0; j < 32; ++j) {
                const float e = (c * 32 + j < T) ? exp2f(fmaf(v[j], sl2, -off)) : 0.f;
                v[j] = e;
                sum += e;
            }
#pragma unroll
            for (int u = 0; u < 4; ++u) {
                uint4 w;
                w.x = pack2(v[8 * u], v[8 * u + 1]);
                w.y = pack2(v[8 * u + 2], v[8 * u + 3]);
                w.z = pack2(v[8 * u + 4], v[8 * u + 5]);
                w.w = pack2(v[8 * u + 6], v[8 * u + 7]);
                *reinterpret_cast<uint4 *>(sP + p_off(r, c * 32 + 8 * u)) = w;
            }
        }
        ptx::fence_proxy_async_smem();
        ptx::tc_fence_before();
        __syncwarp();
        if (lane == 0) ptx::mbar_arrive(bar_p);
        const float inv = 1.f / sum;
        ptx::mbar_wait(bar_o, 0);
        ptx::tc_fence_after();
        float o0[32], o1[32];
        ptx::tmem_ld32(trow, o0);
        ptx::tmem_ld32(trow + 32, o1);
        if (t < T) {
            uint4 *dst = reinterpret_cast<uint4 *>(a.o + (int64_t(b) * T + t) * a.o_ld + h * 64);
#pragma unroll
            for (int u = 0; u < 8; ++u) {
                const float *sv = u < 4 ? o0 + 8 * u : o1 + 8 * (u - 4);
                uint4 w;
                w.x = pack2(sv[0] * inv, sv[1] * inv);
                w.y = pack2(sv[2] * inv, sv[3] * inv);
                w.z = pack2(sv[4] * inv, sv[5] * inv);
                w.w = pack2(sv[6] * inv, sv[7] * inv);
                dst[u] = w;
            }
            a.lse[(int64_t(b) * a.H + h) * T + t] = mx * a.scale + logf(sum);
        }
    }
    ptx::tc_fence_before();
    __syncthreads();
    if (warp == 2) ptx::tmem_dealloc<256>(tmem);
}

// ---------------------------------------------------------------- backward
// Per query tile: S = Q K^T -> P = exp(scale S - lse) (smem, bf16) -> dV += P^T dO, dP = dO V^T ->
// dS = scale P (dP - D), D = rowsum(dO * O) (smem, in place of P) -> dQ = dS K (stored), dK += dS^T Q.
// TMEM (512 columns): [0, 256) S / dP / dQ, [256, 384) dV (two 128-key M tiles), [384, 512) dK.
__global__ void __launch_bounds__(kAttnThreads, 1) attn_bwd_kernel(const __grid_constant__ AttnMaps maps, const AttnArgs a) {
    using namespace attn;
    extern __shared__ __align__(16) uint8_t smem_raw[];
    uint8_t *smem = align1024(smem_raw);
    uint8_t *sQ = smem, *sO = smem + 16384, *sK = smem + 32768, *sV = smem + 65536, *sP = smem + 98304;
    uint64_t *bars = reinterpret_cast<uint64_t *>(smem + 163840);
    uint64_t *bar_kv = bars, *bar_q = bars + 1, *bar_s = bars + 2, *bar_p = bars + 3, *bar_dp = bars + 4,
             *bar_ds = bars + 5, *bar_dq = bars + 6, *bar_free = bars + 7;
    uint32_t *tmem_slot = reinterpret_cast<uint32_t *>(bars + 8);
    const int warp = int(ptx::warp_id()), lane = int(ptx::lane_id());
    const int h = int(blockIdx.x) % a.H, b = int(blockIdx.x) / a.H;
    const int T = a.T, ntile = (T + 127) / 128, nmt = (T + 127) / 128;  // query tiles, key M tiles
    if (warp == 0 && lane == 0) {
        ptx::tma_prefetch_desc(&maps.q);
        ptx::tma_prefetch_desc(&maps.k);
        ptx::tma_prefetch_desc(&maps.v);
        ptx::tma_prefetch_desc(&maps.dout);
    }
    if (warp == 1 && lane == 0) {
        ptx::mbar_init(bar_kv, 1);
        ptx::mbar_init(bar_q, 1);
        ptx::mbar_init(bar_s, 1);
        ptx::mbar_init(bar_p, 4);
        ptx::mbar_init(bar_dp, 1);
        ptx::mbar_init(bar_ds, 4);
        ptx::mbar_init(bar_dq, 1);
        ptx::mbar_init(bar_free, 4);
        ptx::fence_barrier_init();
    }
    if (warp == 2) ptx::tmem_alloc<512>(tmem_slot);
    ptx::tc_fence_before();
    __syncthreads();
    ptx::tc_fence_after();
    const uint32_t tmem = *tmem_slot;
    ptx::griddep_wait();
    ptx::griddep_launch();
    if (warp == 0) {
        if (lane == 0) {
            ptx::mbar_arrive_expect_tx(bar_kv, 65536);
            ptx::tma_load_4d(sK, &maps.k, bar_kv, 0, 0, h, b);
            ptx::tma_load_4d(sV, &maps.v, bar_kv, 0, 0, h, b);
            for (int i = 0; i < ntile; ++i) {
                if (i > 0) ptx::mbar_wait(bar_dq, (i - 1) & 1);  // the previous tile's MMAs read Q / dO
                ptx::mbar_arrive_expect_tx(bar_q, 32768);
                ptx::tma_load_4d(sQ, &maps.q, bar_q, 0, i * 128, h, b);
                ptx::tma_load_4d(sO, &maps.dout, bar_q, 0, i * 128, h, b);
            }
        }
    } else if (warp == 1) {
        if (lane == 0) {
            const uint32_t qa = ptx::smem_u32(sQ), oa = ptx::smem_u32(sO), ka = ptx::smem_u32(sK),
                           va = ptx::smem_u32(sV), pa = ptx::smem_u32(sP);
            const int ksteps = (T + 15) / 16;
            ptx::mbar_wait(bar_kv, 0);
            for (int i = 0; i < ntile; ++i) {
                ptx::mbar_wait(bar_q, i & 1);
                if (i > 0) ptx::mbar_wait(bar_free, (i - 1) & 1);  // dQ of the previous tile drained
                ptx::tc_fence_after();
#pragma unroll
                for (int k = 0; k < 4; ++k) ptx::umma<0>(tmem, desc_k(qa + k * 32), desc_k(ka + k * 32), kIdS, k > 0);
                ptx::umma_commit(bar_s);
                ptx::mbar_wait(bar_p, i & 1);
                ptx::tc_fence_after();
                for (int mt = 0; mt < nmt; ++mt)  // dV[keys] += P^T dO over this tile's 128 queries
#pragma unroll
                    for (int k = 0; k < 8; ++k)
                        ptx::umma<0>(tmem + 256 + mt * 64, desc_mn(pa + mt * 32768 + k * 2048, 16384),
                                     desc_mn(oa + k * 2048, 16384), kIdT, (i > 0 || k > 0) ? 1u : 0u);
#pragma unroll
                for (int k = 0; k < 4; ++k) ptx::umma<0>(tmem, desc_k(oa + k * 32), desc_k(va + k * 32), kIdS, k > 0);
                ptx::umma_commit(bar_dp);
                ptx::mbar_wait(bar_ds, i & 1);
                ptx::tc_fence_after();
                for (int k = 0; k < ksteps; ++k)  // dQ = dS K over the keys
                    ptx::umma<0>(tmem, desc_k(pa + (k >> 2) * 16384 + (k & 3) * 32), desc_mn(ka + k * 2048, 8192),
                                 kIdO, k > 0);
                for (int mt = 0; mt < nmt; ++mt)  // dK[keys] += dS^T Q
#pragma unroll
                    for (int k = 0; k < 8; ++k)
                        ptx::umma<0>(tmem + 384 + mt * 64, desc_mn(pa + mt * 32768 + k * 2048, 16384),
                                     desc_mn(qa + k * 2048, 16384), kIdT, (i > 0 || k > 0) ? 1u : 0u);
                ptx::umma_commit(bar_dq);
            }
        }
    } else if (warp >= 4) {
        const int q = warp & 3, r = q * 32 + lane;
        const uint32_t trow = tmem + (uint32_t(q * 32) << 16);
        const float sl2 = a.scale * kLog2e;
        for (int i = 0; i < ntile; ++i) {
            const int t = i * 128 + r;
            const bool valid = t < T;
            const float lse2 = valid ? a.lse[(int64_t(b) * a.H + h) * T + t] * kLog2e : 0.f;
            ptx::mbar_wait(bar_q, i & 1);  // dO of this tile is in shared memory (TMA writes visible)
            ptx::mbar_wait(bar_s, i & 1);
            // D = rowsum(dO * O): dO from the swizzled tile, O from HBM
            float D = 0.f;
            if (valid) {
                const uint4 *orow = reinterpret_cast<const uint4 *>(a.o + (int64_t(b) * T + t) * a.o_ld + h * 64);
#pragma unroll
                for (int u = 0; u < 8; ++u) {
                    const uint4 ov = orow[u];
                    const uint4 gv = *reinterpret_cast<const uint4 *>(sO + r * 128 + ((u ^ (r & 7)) << 4));
                    const uint32_t ow[4] = {ov.x, ov.y, ov.z, ov.w}, gw[4] = {gv.x, gv.y, gv.z, gv.w};
#pragma unroll
                    for (int e = 0; e < 4; ++e)
                        D = fmaf(bf_lo(gw[e]), bf_lo(ow[e]), fmaf(bf_hi(gw[e]), bf_hi(ow[e]), D));
                }
            }
            ptx::tc_fence_after();
#pragma unroll 1
            for (int c = 0; c < 8; ++c) {  // P = exp(scale S - lse), zero past T and for rows past T
                float v[32];
                if (c * 32 < T) ptx::tmem_ld32(trow + c * 32, v);
#pragma unroll
                for (int j = 0; j < 32; ++j) v[j] = (valid && c * 32 + j < T) ? exp2f(fmaf(v[j], sl2, -lse2)) : 0.f;
#pragma unroll
                for (int u = 0; u < 4; ++u) {
                    uint4 w;
                    w.x = pack2(v[8 * u], v[8 * u + 1]);
                    w.y = pack2(v[8 * u + 2], v[8 * u + 3]);
                    w.z = pack2(v[8 * u + 4], v[8 * u + 5]);
                    w.w = pack2(v[8 * u + 6], v[8 * u + 7]);
                    *reinterpret_cast<uint4 *>(sP + p_off(r, c * 32 + 8 * u)) = w;
                }
            }
            ptx::fence_proxy_async_smem();
            ptx::tc_fence_before();
            __syncwarp();
            if (lane == 0) ptx::mbar_arrive(bar_p);
            ptx::mbar_wait(bar_dp, i & 1);  // dV consumed P; dP is in TMEM
            ptx::tc_fence_after();
#pragma unroll 1
            for (int c = 0; c * 32 < T; ++c) {  // dS = scale P (dP - D), over P in place
                float v[32];
                ptx::tmem_ld32(trow + c * 32, v);
#pragma unroll
                for (int u = 0; u < 4; ++u) {
                    uint4 *pp = reinterpret_cast<uint4 *>(sP + p_off(r, c * 32 + 8 * u));
                    const uint4 pw = *pp;
                    const uint32_t w4[4] = {pw.x, pw.y, pw.z, pw.w};
                    uint32_t o4[4];
#pragma unroll
                    for (int e = 0; e < 4; ++e) {
                        const float d0 = a.scale * bf_lo(w4[e]) * (v[8 * u + 2 * e] - D);
                        const float d1 = a.scale * bf_hi(w4[e]) * (v[8 * u + 2 * e + 1] - D);
                        o4[e] = pack2(d0, d1);
                    }
                    *pp = make_uint4(o4[0], o4[1], o4[2], o4[3]);
                }
            }
            ptx::fence_proxy_async_smem();
            ptx::tc_fence_before();
            __syncwarp();
            if (lane == 0) ptx::mbar_arrive(bar_ds);
            ptx::mbar_wait(bar_dq, i & 1);
            ptx::tc_fence_after();
            float g0[32], g1[32];
            ptx::tmem_ld32(trow, g0);
            ptx::tmem_ld32(trow + 32, g1);
            if (valid) {
                uint4 *dst = reinterpret_cast<uint4 *>(a.dqkv + (int64_t(b) * T + t) * a.dqkv_ld + h * 64);
#pragma unroll
                for (int u = 0; u < 8; ++u) {
                    const float *s = u < 4 ? g0 + 8 * u : g1 + 8 * (u - 4);
                    dst[u] = make_uint4(pack2(s[0], s[1]), pack2(s[2], s[3]), pack2(s[4], s[5]), pack2(s[6], s[7]));
                }
            }
            ptx::tc_fence_before();
            __syncwarp();
            if (lane == 0) ptx::mbar_arrive(bar_free);
        }
        // dV / dK of every key (the last tile's bar_dq covered all their MMAs)
        ptx::tc_fence_after();
        for (int mt = 0; mt < nmt; ++mt) {
            const int key = mt * 128 + r;
#pragma unroll 1
            for (int which = 0; which < 2; ++which) {  // 0: dV, 1: dK
                float g0[32], g1[32];
                const uint32_t col = uint32_t(which == 0 ? 256 : 384) + uint32_t(mt * 64);
                ptx::tmem_ld32(trow + col, g0);
                ptx::tmem_ld32(trow + col + 32, g1);
                if (key < T) {
                    uint4 *dst = reinterpret_cast<uint4 *>(a.dqkv + (int64_t(b) * T + key) * a.dqkv_ld +
                                                           (which == 0 ? a.dv_off : a.dk_off) + h * 64);
#pragma unroll
                    for (int u = 0; u < 8; ++u) {
                        const float *s = u < 4 ? g0 + 8 * u : g1 + 8 * (u - 4);
                        dst[u] = make_uint4(pack2(s[0], s[1]), pack2(s[2], s[3]), pack2(s[4], s[5]), pack2(s[6], s[7]));
                    }
                }
            }
        }
    }
    ptx::tc_fence_before();
    __syncthreads();
    if (warp == 2) ptx::tmem_dealloc<512>(tmem);
}

}  // namespace cdp
