// tcgen05 / TMEM / TMA GEMM for sm_100a with pluggable fused epilogues.
//
//   D[M,N] (fp32, in TMEM) = sum_seg A_seg[M,K] . B_seg[K,N]
//
// * one 128 x BN output tile per CTA (cta_group::1, UMMA M=128), split-K over
//   gridDim.z with a deterministic in-order fix-up by the last-arriving CTA;
// * operands staged by TMA into 128-byte-swizzled shared memory, a STAGES-deep
//   mbarrier ring between the TMA warp (warp 0) and the single MMA-issuing
//   thread (warp 1); warp 2 owns the TMEM allocation; warps 4-7 are the
//   epilogue (thread t <-> accumulator row t, tcgen05.ld 32 columns at a time);
// * A and B may each be K-major or MN-major (the instruction descriptor's
//   transpose bits), so row-major activations [samples, features] and the
//   row-major weights [din, dout] of the reference layout feed all three
//   GEMMs of a layer (forward, weight-grad, data-grad) without transposes;
// * KIND 0: bf16 operands (kind::f16). KIND 1: fp32 operands read as tf32
//   (kind::tf32); three segments (hi.hi + hi.lo + lo.hi) give the 3xTF32
//   fp32-accurate product used by the fp32 parity mode.
#pragma once
#include "ptx.cuh"

namespace cdp {

struct GemmMaps {
    CUtensorMap a[3];
    CUtensorMap b[3];
    CUtensorMap o;  // output tile map of the TMA-store epilogue (gemm_pk_kernel, PkArgs::tma_out)
    CUtensorMap e[2];  // epilogue operand maps (residual gradient, mask) of a kTmaAdd epilogue
};

// Implicit-GEMM convolution geometry (MODE 1-3 of gemm_tc_kernel).  Pixels
// are tiled in boxes (bw x bh x bn) of a [Bn][Ho][Wo] grid; one box is one
// 4-D TMA load (channels innermost) of an NHWC tensor, with element strides
// for strided convolutions and out-of-bounds zero fill as the padding.
struct ConvGeom {
    int C;              // channels of the gathered NHWC tensor
    int R, S, stride, pad;
    int cpt;            // CH-channel chunks per filter tap (C / CH)
    int bw, bh, bn;     // pixel box (output space; dgrad: input space)
    int nbw, nbh;       // boxes along W and H
    int Wo, Ho, Bn;     // extents of the boxed pixel grid
    int Cw;             // dgrad: Cin (rows per tap of W viewed [R*S*Cin][Cout])
    // dgrad taps: A box offset (toh, tow) on dy and weight tap twt (= r*S + s) of tap k;
    // a stride-2 data gradient runs as 4 sub-pixel phases, each with its own tap subset
    int ntap;
    signed char toh[9], tow[9], twt[9];
    // output row of grid pixel (b, h, w): (b*oH + h*omul + oph)*oW + w*omul + opw
    int omul, oph, opw, oH, oW;
};

__host__ __device__ inline void conv_box_origin(const ConvGeom &g, int idx, int &w0, int &h0, int &b0) {
    const int iw = idx % g.nbw;
    const int t = idx / g.nbw;
    const int ih = t % g.nbh;
    w0 = iw * g.bw;
    h0 = ih * g.bh;
    b0 = (t / g.nbh) * g.bn;
}

// Row `row` of box `idx` -> flat pixel index (b*Ho + h)*Wo + w, or -1 outside the grid.
__host__ __device__ inline int conv_box_row(const ConvGeom &g, int idx, int row) {
    int w0, h0, b0;
    conv_box_origin(g, idx, w0, h0, b0);
    const int w = w0 + row % g.bw, h = h0 + (row / g.bw) % g.bh, b = b0 + row / (g.bw * g.bh);
    if (w >= g.Wo || h >= g.Ho || b >= g.Bn) return -1;
    const int oh = h * g.omul + g.oph, ow = w * g.omul + g.opw;
    if (oh >= g.oH || ow >= g.oW) return -1;  // a phase pixel past an odd input edge
    return (b * g.oH + oh) * g.oW + ow;
}

struct GemmArgs {
    int M, N;
    int kb_per_seg;   // k-blocks (of 128 bytes of K) per segment
    int n_seg;        // 1..3
    int iters_per_split;
    float *ws;        // split-K partials [tiles][splits][128][BN]
    int *counters;    // per tile arrival counters (self-resetting)
    ConvGeom cv;      // MODE 1-3 only
};

// GM_BATCH: independent GEMMs over a (head, sample) grid, every operand a 4-D TMA view
// {inner, rows, heads, samples} of a token-major buffer (attention score / value products).
enum GemmMode { GM_PLAIN = 0, GM_FPROP = 1, GM_DGRAD = 2, GM_WGRAD = 3, GM_BATCH = 4 };

template <int KIND, int BN_, bool A_MN, bool B_MN, int ST = 0, int PF = 0>
struct GemmCfg {
    static constexpr int BM = 128;
    static constexpr int BN = BN_;
    static constexpr int ELEM = KIND == 0 ? 2 : 4;
    static constexpr int BK = 128 / ELEM;      // K elements per k-block
    static constexpr int UMMA_K = 32 / ELEM;   // K per tcgen05.mma
    static constexpr int CH = 128 / ELEM;      // MN elements per 128-byte swizzle row
    static constexpr int A_BYTES = BM * 128;
    static constexpr int B_BYTES = BN * 128;
    static constexpr int STAGE_BYTES = A_BYTES + B_BYTES;
    static constexpr int STAGES = ST ? ST : ((200 * 1024 / STAGE_BYTES) > 6 ? 6 : (200 * 1024 / STAGE_BYTES));
    static constexpr int PF_BYTES = PF;  // epilogue prefetch area (after the operand ring)
    static constexpr uint32_t TMEM_COLS = BN <= 32 ? 32 : BN <= 64 ? 64 : BN <= 128 ? 128 : 256;
    static constexpr int SMEM = 1024 + STAGES * STAGE_BYTES + PF_BYTES + 256;
    static constexpr uint32_t IDESC = ptx::instr_desc(KIND == 0 ? 1u : 2u, A_MN, B_MN, 128, BN);
    static_assert(BN % 32 == 0 && BN >= 32 && BN <= 256, "BN must be a multiple of 32 in [32,256]");
    static_assert(!B_MN || BN % CH == 0, "MN-major B needs BN multiple of the 128-byte row");
    static_assert(STAGES >= 2, "not enough shared memory for two stages");
};

// Load one k-block of a 128-row (A) or BN-row (B) operand tile.
template <class C, bool MN, int ROWS>
__device__ __forceinline__ void load_operand(uint8_t *dst, const CUtensorMap *m, uint64_t *bar, int mn0, int k0) {
    if constexpr (!MN) {
        ptx::tma_load_2d(dst, m, bar, k0, mn0);  // tensor (inner K, outer MN)
    } else {
#pragma unroll
        for (int c = 0; c < ROWS / C::CH; ++c)  // tensor (inner MN, outer K)
            ptx::tma_load_2d(dst + c * (C::BK * 128), m, bar, mn0 + c * C::CH, k0);
    }
}

// Implicit-GEMM convolution producer: the k-block `kb` of segment `seg` for the
// CTA's M tile (box `m_tile` for FPROP / DGRAD, rows m0.. for WGRAD).
//   FPROP: A = input gathered at tap (r,s) (box shifted by r-pad, s-pad, strided),
//          B = weights [R*S*C][Cout] (MN-major), k-block = one CH-channel chunk of a tap;
//   DGRAD: (stride 1) A = dy gathered at (pad-r, pad-s), B = W^T: rows tap*Cin + n of
//          W viewed [R*S*Cin][Cout] (K-major);
//   WGRAD: M = (tap, c), K = pixels: A = input gathered per 64-row chunk at its tap
//          (MN-major), B = dy (MN-major), k-block = one pixel box.
// B operand of a CTA pair (CL = 2, MN-major B only): each CTA loads every other
// 128-byte column chunk of the B tile and multicasts it to both CTAs.
template <class C, bool MN, int BN, int CL>
__device__ __forceinline__ void load_b(uint8_t *dst, const CUtensorMap *m, uint64_t *bar, int n0, int k0, int rank) {
    if constexpr (CL == 1) {
        (void)rank;
        load_operand<C, MN, BN>(dst, m, bar, n0, k0);
    } else {
        static_assert(MN && BN / C::CH >= 2, "paired B loads need an MN-major B of at least two chunks");
#pragma unroll
        for (int c = 0; c < BN / C::CH; ++c)
            if ((c & 1) == rank) ptx::tma_load_2d_mc(dst + c * (C::BK * 128), m, bar, n0 + c * C::CH, k0, 3);
    }
}

template <class C, int MODE, bool B_MN, int BN, int CL = 1>
__device__ __forceinline__ void conv_load(uint8_t *sa, uint8_t *sb, const GemmMaps &maps, const ConvGeom &g,
                                          uint64_t *bar, int seg, int kb, int m_tile, int m0, int n0, int rank = 0) {
    static_assert(CL == 1 || (MODE != GM_DGRAD && B_MN && BN / C::CH >= 2), "paired B loads need an MN-major B");
    if constexpr (MODE == GM_FPROP || MODE == GM_DGRAD) {
        const int tap = kb / g.cpt, cc = kb - tap * g.cpt;
        const int r = tap / g.S, s = tap - r * g.S;
        int w0, h0, b0;
        conv_box_origin(g, m_tile, w0, h0, b0);
        if constexpr (MODE == GM_FPROP) {
            ptx::tma_load_4d(sa, &maps.a[seg], bar, cc * C::CH, w0 * g.stride - g.pad + s, h0 * g.stride - g.pad + r,
                             b0);
            load_b<C, B_MN, BN, CL>(sb, &maps.b[seg], bar, n0, kb * C::BK, rank);
        } else {
            (void)r;
            (void)s;
            ptx::tma_load_4d(sa, &maps.a[seg], bar, cc * C::CH, w0 + g.tow[tap], h0 + g.toh[tap], b0);
            ptx::tma_load_2d(sb, &maps.b[seg], bar, cc * C::CH, g.twt[tap] * g.Cw + n0);
        }
    } else {
        int w0, h0, b0;
        conv_box_origin(g, kb, w0, h0, b0);
        const int taps = g.R * g.S;
#pragma unroll
        for (int q = 0; q < 128 / C::CH; ++q) {
            const int mrow = m0 + q * C::CH;
            const int tap = min(mrow / g.C, taps - 1);
            const int c0 = mrow - (mrow / g.C) * g.C;
            const int r = tap / g.S, s = tap - r * g.S;
            ptx::tma_load_4d(sa + q * (C::BK * 128), &maps.a[seg], bar, c0, w0 * g.stride - g.pad + s,
                             h0 * g.stride - g.pad + r, b0);
        }
#pragma unroll
        for (int q = 0; q < BN / C::CH; ++q) {
            if constexpr (CL == 1)
                ptx::tma_load_4d(sb + q * (C::BK * 128), &maps.b[seg], bar, n0 + q * C::CH, w0, h0, b0);
            else if ((q & 1) == rank)
                ptx::tma_load_4d_mc(sb + q * (C::BK * 128), &maps.b[seg], bar, n0 + q * C::CH, w0, h0, b0, 3);
        }
    }
}

// Producer-side iterator over the k-blocks of one unit of the persistent kernel
// (gemm_pk_kernel): the same loads as conv_load, with the per-unit geometry
// hoisted and the per-k-block indices advanced by counters instead of integer
// division (the single producer thread's address arithmetic was the mainloop's
// critical path for the implicit-conv modes).
template <class C, int MODE>
struct ConvIter {
    static constexpr int NQ = 128 / C::CH;  // 128-byte column chunks of the 128-row A tile (WGRAD)
    int seg, kb, kb_per_seg;
    int tap, cc, r, s;  // FPROP / DGRAD: k-block = (tap, channel chunk)
    int w0, h0, b0;     // FPROP / DGRAD: the M tile's pixel box; WGRAD: the k-block's pixel box
    int iw, ih;         // WGRAD: pixel box counters
    int qc[NQ], qs[NQ], qr[NQ];  // WGRAD: channel / tap (s, r) of each A chunk

    __device__ __forceinline__ void init(const ConvGeom &g, int kbps, int lo, int m_tile, int m0) {
        kb_per_seg = kbps;
        seg = lo / kbps;
        kb = lo - seg * kbps;
        if constexpr (MODE == GM_FPROP || MODE == GM_DGRAD) {
            tap = kb / g.cpt;
            cc = kb - tap * g.cpt;
            r = tap / g.S;
            s = tap - r * g.S;
            conv_box_origin(g, m_tile, w0, h0, b0);
        } else if constexpr (MODE == GM_WGRAD) {
            iw = kb % g.nbw;
            const int t = kb / g.nbw;
            ih = t % g.nbh;
            b0 = (t / g.nbh) * g.bn;
            w0 = iw * g.bw;
            h0 = ih * g.bh;
            const int taps = g.R * g.S;
#pragma unroll
            for (int q = 0; q < NQ; ++q) {
                const int mrow = m0 + q * C::CH;
                const int tq = min(mrow / g.C, taps - 1);
                qc[q] = mrow - (mrow / g.C) * g.C;
                qr[q] = tq / g.S;
                qs[q] = tq - qr[q] * g.S;
            }
        }
    }
    __device__ __forceinline__ void next(const ConvGeom &g) {
        if (++kb == kb_per_seg) {  // next 3xTF32 segment: restart the k sequence
            kb = 0;
            ++seg;
            if constexpr (MODE == GM_FPROP || MODE == GM_DGRAD) {
                tap = cc = r = s = 0;
            } else if constexpr (MODE == GM_WGRAD) {
                iw = ih = 0;
                w0 = h0 = b0 = 0;
            }
            return;
        }
        if constexpr (MODE == GM_FPROP || MODE == GM_DGRAD) {
            if (++cc == g.cpt) {
                cc = 0;
                ++tap;
                if (++s == g.S) {
                    s = 0;
                    ++r;
                }
            }
        } else if constexpr (MODE == GM_WGRAD) {
            if (++iw == g.nbw) {
                iw = 0;
                w0 = 0;
                if (++ih == g.nbh) {
                    ih = 0;
                    h0 = 0;
                    b0 += g.bn;
                } else {
                    h0 += g.bh;
                }
            } else {
                w0 += g.bw;
            }
        }
    }
    // Issue the k-block's loads (A, and the CL-shared B) onto `bar`.
    template <bool B_MN, int BN, int CL>
    __device__ __forceinline__ void load(uint8_t *sa, uint8_t *sb, const GemmMaps &maps, const ConvGeom &g,
                                         uint64_t *bar, int n0, int rank) const {
        if constexpr (MODE == GM_FPROP) {
            ptx::tma_load_4d(sa, &maps.a[seg], bar, cc * C::CH, w0 * g.stride - g.pad + s, h0 * g.stride - g.pad + r,
                             b0);
            load_b<C, B_MN, BN, CL>(sb, &maps.b[seg], bar, n0, kb * C::BK, rank);
        } else if constexpr (MODE == GM_DGRAD) {
            static_assert(CL == 1, "paired B loads need an MN-major B");
            ptx::tma_load_4d(sa, &maps.a[seg], bar, cc * C::CH, w0 + g.tow[tap], h0 + g.toh[tap], b0);
            ptx::tma_load_2d(sb, &maps.b[seg], bar, cc * C::CH, g.twt[tap] * g.Cw + n0);
        } else {
#pragma unroll
            for (int q = 0; q < NQ; ++q)
                ptx::tma_load_4d(sa + q * (C::BK * 128), &maps.a[seg], bar, qc[q], w0 * g.stride - g.pad + qs[q],
                                 h0 * g.stride - g.pad + qr[q], b0);
#pragma unroll
            for (int q = 0; q < BN / C::CH; ++q) {
                if constexpr (CL == 1)
                    ptx::tma_load_4d(sb + q * (C::BK * 128), &maps.b[seg], bar, n0 + q * C::CH, w0, h0, b0);
                else if ((q & 1) == rank)
                    ptx::tma_load_4d_mc(sb + q * (C::BK * 128), &maps.b[seg], bar, n0 + q * C::CH, w0, h0, b0, 3);
            }
        }
    }
};

template <class C, bool MN>
__device__ __forceinline__ uint64_t operand_desc(uint32_t base, int k) {
    if constexpr (!MN)
        return ptx::smem_desc_sw128(base + k * 32, 16, 1024);
    else if constexpr (C::ELEM == 2)
        return ptx::smem_desc_sw128(base + k * C::UMMA_K * 128, C::BK * 128, 1024);
    else  // tf32 MN-major: 32-byte swizzle atoms, 4-row groups
        return ptx::smem_desc_sw128(base + k * C::UMMA_K * 128, C::BK * 128, 512, 1);
}

template <int KIND, int BN, bool A_MN, bool B_MN, class Epi, int MODE = GM_PLAIN>
__global__ void __launch_bounds__(256, 1)
    gemm_tc_kernel(const __grid_constant__ GemmMaps maps, const GemmArgs args, const typename Epi::Params ep) {
    using C = GemmCfg<KIND, BN, A_MN, B_MN, Epi::kStages, Epi::template pf_bytes<BN>()>;
    extern __shared__ __align__(16) uint8_t smem_raw[];
    uint8_t *smem = smem_raw + ((1024u - (ptx::smem_u32(smem_raw) & 1023u)) & 1023u);
    uint8_t *sA = smem;
    uint8_t *sB = smem + C::STAGES * C::A_BYTES;
    float *pf = reinterpret_cast<float *>(smem + C::STAGES * C::STAGE_BYTES);
    uint64_t *full = reinterpret_cast<uint64_t *>(smem + C::STAGES * C::STAGE_BYTES + C::PF_BYTES);
    uint64_t *empty = full + C::STAGES;
    uint64_t *tmem_full = empty + C::STAGES;
    uint32_t *tmem_slot = reinterpret_cast<uint32_t *>(tmem_full + 1);
    int *last_flag = reinterpret_cast<int *>(tmem_slot + 1);

    const uint32_t warp = ptx::warp_id();
    const int m0 = blockIdx.x * C::BM;
    const int n0 = blockIdx.y * BN;
    const int split = blockIdx.z;
    const int total_iters = args.kb_per_seg * args.n_seg;
    const int it_lo = split * args.iters_per_split;
    const int it_hi = min(total_iters, it_lo + args.iters_per_split);
    const int n_iters = it_hi - it_lo;

    if (warp == 0 && ptx::lane_id() == 0) {
        for (int s = 0; s < args.n_seg; ++s) {
            ptx::tma_prefetch_desc(&maps.a[s]);
            ptx::tma_prefetch_desc(&maps.b[s]);
        }
    }
    if (warp == 1 && ptx::lane_id() == 0) {
        for (int s = 0; s < C::STAGES; ++s) {
            ptx::mbar_init(&full[s], 1);
            ptx::mbar_init(&empty[s], 1);
        }
        ptx::mbar_init(tmem_full, 1);
        ptx::fence_barrier_init();
    }
    if (warp == 2) ptx::tmem_alloc<C::TMEM_COLS>(tmem_slot);
    ptx::tc_fence_before();
    __syncthreads();
    ptx::tc_fence_after();
    const uint32_t tmem_base = *tmem_slot;
    // PDL: the prologue above overlapped the previous kernel; global memory is
    // touched only after the predecessor's results are visible.
    ptx::griddep_wait();
    ptx::griddep_launch();

    if (warp == 0) {
        if (ptx::lane_id() == 0) {
            for (int it = 0; it < n_iters; ++it) {
                const int s = it % C::STAGES;
                if (it >= C::STAGES) ptx::mbar_wait(&empty[s], ((it / C::STAGES) - 1) & 1);
                const int g = it_lo + it;
                const int seg = g / args.kb_per_seg;
                const int k0 = (g % args.kb_per_seg) * C::BK;
                ptx::mbar_arrive_expect_tx(&full[s], C::STAGE_BYTES);
                if constexpr (MODE == GM_PLAIN) {
                    load_operand<C, A_MN, 128>(sA + s * C::A_BYTES, &maps.a[seg], &full[s], m0, k0);
                    load_operand<C, B_MN, BN>(sB + s * C::B_BYTES, &maps.b[seg], &full[s], n0, k0);
                } else {
                    conv_load<C, MODE, B_MN, BN>(sA + s * C::A_BYTES, sB + s * C::B_BYTES, maps, args.cv, &full[s],
                                                 seg, g % args.kb_per_seg, blockIdx.x, m0, n0);
                }
            }
        }
    } else if (warp == 1) {
        if (ptx::lane_id() == 0) {
            for (int it = 0; it < n_iters; ++it) {
                const int s = it % C::STAGES;
                ptx::mbar_wait(&full[s], (it / C::STAGES) & 1);
                ptx::tc_fence_after();
                const uint32_t a_base = ptx::smem_u32(sA + s * C::A_BYTES);
                const uint32_t b_base = ptx::smem_u32(sB + s * C::B_BYTES);
#pragma unroll
                for (int k = 0; k < C::BK / C::UMMA_K; ++k) {
                    ptx::umma<KIND>(tmem_base, operand_desc<C, A_MN>(a_base, k), operand_desc<C, B_MN>(b_base, k),
                                    C::IDESC, (it > 0 || k > 0) ? 1u : 0u);
                }
                ptx::umma_commit(&empty[s]);
            }
            ptx::umma_commit(tmem_full);
        }
    } else if (warp >= 4 && !Epi::kTile) {
        // ---- per-row epilogue: thread t of warps 4-7 owns accumulator row t
        const int q = warp - 4;  // TMEM lane quarter of this warp
        const int row = q * 32 + ptx::lane_id();
        int m = m0 + row;
        if constexpr (MODE == GM_FPROP || MODE == GM_DGRAD) {
            m = conv_box_row(args.cv, blockIdx.x, row);
            if (m < 0) m = args.M;  // outside the pixel grid: the epilogue skips rows >= M
        }
        const uint32_t taddr = tmem_base + (uint32_t(q * 32) << 16);
        ptx::mbar_wait(tmem_full, 0);
        ptx::tc_fence_after();
        typename Epi::State st;
        if (gridDim.z == 1) {
            Epi::begin(ep, m, st);
#pragma unroll 1
            for (int c = 0; c < BN; c += 32) {
                float v[32];
                ptx::tmem_ld32(taddr + c, v);
                if (n_iters == 0) {
#pragma unroll
                    for (int i = 0; i < 32; ++i) v[i] = 0.f;
                }
                Epi::apply(ep, m, n0 + c, v, args.M, args.N, st);
            }
            Epi::finish(ep, m, args.M, st);
            if (blockIdx.x == 0 && blockIdx.y == 0) Epi::extra(ep, threadIdx.x - 128, 128);
        } else {
            const int tile = blockIdx.y * gridDim.x + blockIdx.x;
            float *mine = args.ws + ((size_t(tile) * gridDim.z + split) * 128 + row) * BN;
#pragma unroll 1
            for (int c = 0; c < BN; c += 32) {
                float v[32];
                ptx::tmem_ld32(taddr + c, v);
#pragma unroll
                for (int i = 0; i < 32; i += 4)
                    *reinterpret_cast<float4 *>(mine + c + i) = make_float4(v[i], v[i + 1], v[i + 2], v[i + 3]);
            }
            __threadfence();
            asm volatile("bar.sync 1, 128;" ::: "memory");
            if (threadIdx.x == 128) {
                const int prev = atomicAdd(&args.counters[tile], 1);
                const int last = prev == int(gridDim.z) - 1;
                if (last) args.counters[tile] = 0;
                *last_flag = last;
            }
            asm volatile("bar.sync 1, 128;" ::: "memory");
            if (*last_flag) {
                __threadfence();
                const float *base = args.ws + (size_t(tile) * gridDim.z * 128 + row) * BN;
                Epi::begin(ep, m, st);
#pragma unroll 1
                for (int c = 0; c < BN; c += 32) {
                    float v[32];
#pragma unroll
                    for (int i = 0; i < 32; ++i) v[i] = 0.f;
#pragma unroll 4
                    for (int z = 0; z < int(gridDim.z); ++z) {
                        const float *p = base + size_t(z) * 128 * BN + c;
#pragma unroll
                        for (int i = 0; i < 32; i += 4) {
                            float4 t = __ldcg(reinterpret_cast<const float4 *>(p + i));
                            v[i] += t.x;
                            v[i + 1] += t.y;
                            v[i + 2] += t.z;
                            v[i + 3] += t.w;
                        }
                    }
                    Epi::apply(ep, m, n0 + c, v, args.M, args.N, st);
                }
                Epi::finish(ep, m, args.M, st);
                if (blockIdx.x == 0 && blockIdx.y == 0) Epi::extra(ep, threadIdx.x - 128, 128);
            }
        }
    }
    if constexpr (Epi::kTile) {
        // ---- tile epilogue: TMEM -> shared (the drained operand ring), then all
        // 256 threads apply the epilogue with coalesced 128-bit global accesses.
        // Split-K: every CTA parks its partial tile in the workspace; the last
        // arriving CTA of the tile sums them in split order and runs the epilogue.
        constexpr int LDS = BN + 4;
        float *stile = reinterpret_cast<float *>(smem);
        const bool split = gridDim.z > 1;
        if (warp >= 4) {
            const int q = warp - 4;
            const int row = q * 32 + ptx::lane_id();
            const uint32_t taddr = tmem_base + (uint32_t(q * 32) << 16);
            // while TMA + MMA run: protocol waits, then prefetch of the epilogue's
            // other operands (parameters, momentum, previous partial) into shared
            Epi::pre(ep, threadIdx.x - 128);
            if (!split) Epi::template prefetch<BN>(ep, pf, m0, n0, args.M, args.N, threadIdx.x - 128, 128);
            ptx::cp_async_commit();
            ptx::mbar_wait(tmem_full, 0);
            ptx::tc_fence_after();
#pragma unroll 1
            for (int c = 0; c < BN; c += 32) {
                float v[32];
                ptx::tmem_ld32(taddr + c, v);
                if (n_iters == 0) {
#pragma unroll
                    for (int i = 0; i < 32; ++i) v[i] = 0.f;
                }
#pragma unroll
                for (int i = 0; i < 32; i += 4)
                    *reinterpret_cast<float4 *>(stile + row * LDS + c + i) = make_float4(v[i], v[i + 1], v[i + 2], v[i + 3]);
            }
            ptx::cp_async_wait_all();
        }
        __syncthreads();
        bool run = true;
        if (split) {
            const int tile = blockIdx.y * gridDim.x + blockIdx.x;
            float *mine = args.ws + (size_t(tile) * gridDim.z + blockIdx.z) * 128 * BN;
            constexpr int C4 = BN / 4;
            for (int e = threadIdx.x; e < 128 * C4; e += blockDim.x) {
                const int r = e / C4, c = (e % C4) * 4;
                *reinterpret_cast<float4 *>(mine + r * BN + c) = *reinterpret_cast<const float4 *>(stile + r * LDS + c);
            }
            __threadfence();
            __syncthreads();
            if (threadIdx.x == 0) {
                const int prev = atomicAdd(&args.counters[tile], 1);
                const int last = prev == int(gridDim.z) - 1;
                if (last) args.counters[tile] = 0;
                *last_flag = last;
            }
            __syncthreads();
            run = *last_flag != 0;
            if (run) {
                __threadfence();
                const float *base = args.ws + size_t(tile) * gridDim.z * 128 * BN;
                for (int e = threadIdx.x; e < 128 * C4; e += blockDim.x) {
                    const int r = e / C4, c = (e % C4) * 4;
                    float4 acc = make_float4(0.f, 0.f, 0.f, 0.f);
                    for (int z = 0; z < int(gridDim.z); ++z) {
                        const float4 t = __ldcg(reinterpret_cast<const float4 *>(base + size_t(z) * 128 * BN + r * BN + c));
                        acc.x += t.x;
                        acc.y += t.y;
                        acc.z += t.z;
                        acc.w += t.w;
                    }
                    *reinterpret_cast<float4 *>(stile + r * LDS + c) = acc;
                }
                __syncthreads();
            }
        }
        if (run) {
            Epi::template tile<BN>(ep, stile, LDS, split ? nullptr : pf, m0, n0, args.M, args.N, threadIdx.x,
                                   blockDim.x);
            if (blockIdx.x == 0 && blockIdx.y == 0) Epi::extra(ep, threadIdx.x, blockDim.x);
            Epi::post(ep, threadIdx.x, gridDim.x * gridDim.y);
        }
    }
    ptx::tc_fence_before();
    __syncthreads();
    if (warp == 2) ptx::tmem_dealloc<C::TMEM_COLS>(tmem_base);
}

}  // namespace cdp
