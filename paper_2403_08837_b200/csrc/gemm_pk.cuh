// Persistent tcgen05 GEMM for sm_100a (the conv / ResNet hot path).
//
//   D[M,N] (fp32, TMEM) = sum_seg A_seg[M,K] . B_seg[K,N], plain or implicit-conv
//   operands (GemmMode, conv_load in gemm.cuh), fused epilogue per output tile.
//
// One CTA per SM loops over work units (tile_m, tile_n, split) with three
// pipelines:
//   * smem ring  : warp 0 (one thread) issues TMA into a STAGES-deep
//                  full/empty mbarrier ring;
//   * TMEM ring  : warp 1 (one thread) issues tcgen05.mma into one of TWO
//                  accumulators (2 x BN columns), so the epilogue of unit j
//                  overlaps the mainloop of unit j+1;
//   * epilogue   : warps 4-11 drain the accumulator (tcgen05.ld; warp w reads
//                  TMEM lane quarter w % 4, column half (w - 4) / 4) into a
//                  padded shared tile, release the accumulator, then run the
//                  fused epilogue on the shared tile with all 256 threads
//                  (coalesced 16-byte global accesses, several in flight each).
// Split-K units write their partial tile to a workspace; a separate kernel
// (pk_reduce_kernel) sums the partials in split order - deterministic and
// parallel over (tile, row chunk) - and runs the same epilogue.
#pragma once
#include <cuda_bf16.h>

#include <cstdlib>
#include <type_traits>

#include "gemm.cuh"
#include "host.h"

namespace cdp {

struct PkArgs {
    int M, N;
    int tiles_m, tiles_n, splits;
    int kb_per_seg, n_seg, iters_per_split, total_iters;
    int units;
    int boxed;     // rows of an M tile are a pixel box of cv (FPROP / DGRAD)
    float *ws;     // split partials [tile][split][128][BN]
    ConvGeom cv;
    // GM_BATCH: nbatch = heads * samples independent GEMMs; batch g = (head g % nh, sample g / nh);
    // the epilogue's output offset of batch g = (g / nh) * out_bs + (g % nh) * out_hs elements
    int nbatch, nh;
    int64_t out_bs, out_hs;
    // CTA pairs (CL = 2): units enumerate (tile-pair, tile_n, split); rank r of the
    // pair takes M tile 2 * pair + r (>= tiles_m: a phantom that only feeds its partner)
    int tiles_pm;
    // TMA-store epilogue (Epi::kTmaStore, non-split units): the tile is converted to bf16 into a
    // 128-byte-swizzled shared staging area in 64-column chunks and written by TMA through maps.o
    // (2-D {N, M} for GM_PLAIN, 4-D {N, W, H, B} with the pixel box for FPROP / stride-1 DGRAD)
    int tma_out;
    // TMA-staged epilogue operands (Epi::kTmaAdd): number of operand maps in GemmMaps::e (1: residual,
    // 2: residual + mask); 2-D {N, M} maps for GM_PLAIN, 4-D {N, W, H, B} pixel-box maps otherwise
    int tma_add;
    // BN statistics of a 128-column TMA-store tile by two tensor-core MMAs (opt-in, CDP_MMA_STATS=1: correct,
    // but slower than the staging read-back on B200 — the MMAs queue behind the next unit's mainloop)
    int mma_stats;
    // Grouped TMA-store epilogue (plain bf16 outputs of unsplit units, CDP_PK_GROUPED=0 disables): epilogue
    // warps 4-7 take the units of accumulator 0, warps 8-11 those of accumulator 1, each group a whole
    // tile with its own staging buffer, barrier and statistics slot (two tiles' epilogues in flight:
    // the one-group-per-tile epilogue left 62 % of issue cycles without an eligible warp)
    int grouped;
    // Stride-2 data gradient with all sub-pixel phases in one launch (nph > 1): the batch index g of
    // a unit is its phase, cvp[g] its geometry (tap table, output phase offsets); no split-K.
    int nph;
    ConvGeom cvp[4];
};

// Epilogues with a direct (register-only) path declare kDirect (EpiConvOut2 bf16).
template <class E, class = void>
struct pk_direct : std::false_type {};
template <class E>
struct pk_direct<E, std::void_t<decltype(E::kDirect)>> : std::bool_constant<E::kDirect> {};

// Epilogues whose extra row operands (residual gradient, mask) are staged into shared memory by TMA
// (warp 3 as their producer) declare kTmaAdd and kEbufSlots (ring slots of 64 columns x 128 rows of
// both operands, 128-byte swizzled: 32 KB each).
template <class E, class = void>
struct pk_tma_add : std::false_type {};
template <class E>
struct pk_tma_add<E, std::void_t<decltype(E::kTmaAdd)>> : std::bool_constant<E::kTmaAdd> {};
template <class E>
constexpr int pk_ebuf_slots() {
    if constexpr (pk_tma_add<E>::value)
        return E::kEbufSlots;
    else
        return 0;
}
template <class E>
constexpr int pk_ebuf_bytes() {
    return pk_ebuf_slots<E>() * 32768;
}

__device__ __forceinline__ const ConvGeom &pk_geom(const PkArgs &a, int g) { return a.nph > 1 ? a.cvp[g] : a.cv; }

template <int KIND, int BN, bool A_MN, bool B_MN, int ST, int EB = 0>
struct PkCfg {
    static constexpr int BM = 128;
    static constexpr int ELEM = KIND == 0 ? 2 : 4;
    static constexpr int BK = 128 / ELEM;
    static constexpr int UMMA_K = 32 / ELEM;
    static constexpr int CH = 128 / ELEM;
    static constexpr int A_BYTES = BM * 128;
    static constexpr int B_BYTES = BN * 128;
    static constexpr int STAGE_BYTES = A_BYTES + B_BYTES;
    static constexpr int EPI_COLS = BN < 128 ? BN : 128;  // columns staged per epilogue pass
    static constexpr int LDS = EPI_COLS + 4;
    static constexpr int STILE_BYTES = 128 * LDS * 4;
    // epilogue region: the fp32 shared tile, or (EB > 0) the TMA-staged epilogue operand ring
    static constexpr int EPI_BYTES = EB > STILE_BYTES ? EB : STILE_BYTES;
    // per TMEM quarter column up to 3 statistics (drain path), or [8 warps][EPI_COLS][2] (TMA-store path)
    static constexpr int PART_BYTES = (4 * EPI_COLS * 3 * 4 > 8 * EPI_COLS * 8) ? 4 * EPI_COLS * 3 * 4 : 8 * EPI_COLS * 8;
    static constexpr int BUDGET = 224 * 1024 - EPI_BYTES - PART_BYTES - 2048;
    static constexpr int STAGES = ST ? ST : (BUDGET / STAGE_BYTES > 8 ? 8 : BUDGET / STAGE_BYTES);
    static constexpr uint32_t TMEM_COLS = 2 * BN <= 32 ? 32 : 2 * BN <= 64 ? 64 : 2 * BN <= 128 ? 128 : 2 * BN <= 256 ? 256 : 512;
    static constexpr int PRE_BYTES = 2 * 128 * 8;  // running column statistics of the unit (cp.async)
    static constexpr int ONES_BYTES = 4096;        // bf16 ones [16][128] (K-major): the column-sum MMA's B
    // rowm 512 B + barriers 256 B + PRE_BYTES, padded to 3 KB so the ones tile starts 1024-aligned
    static constexpr int SMEM = 1024 + STAGES * STAGE_BYTES + EPI_BYTES + PART_BYTES + 3072 + ONES_BYTES;
    static_assert(512 + 256 + PRE_BYTES <= 3072, "rowm / barrier / statistics-slot area");
    static constexpr uint32_t IDESC = ptx::instr_desc(KIND == 0 ? 1u : 2u, A_MN, B_MN, 128, BN);
    static_assert(BN % 64 == 0 && BN >= 64 && BN <= 256, "BN must be 64, 128 or 256");
    static_assert(!B_MN || BN % CH == 0, "MN-major B needs BN multiple of the 128-byte row");
    static_assert(STAGES >= 2, "not enough shared memory for two stages");
    static_assert(SMEM <= 227 * 1024, "shared memory budget exceeded");
};

__device__ __forceinline__ void pk_bar(int id, int n) { asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(n) : "memory"); }

// Column sums of a warp's 32 x 32 block (lane = row, v[i] = column i):
// recursive-halving reduce-scatter, 31 shuffles; lane l returns column l's sum
// over the 32 rows in a fixed order.
__device__ __forceinline__ float warp_colsum32(float (&v)[32]) {
    const int lane = ptx::lane_id();
#pragma unroll
    for (int off = 16; off >= 1; off >>= 1) {
        const bool upper = (lane & off) != 0;
#pragma unroll
        for (int i = 0; i < off; ++i) {
            const float send = upper ? v[i] : v[i + off];
            const float keep = upper ? v[i + off] : v[i];
            v[i] = keep + __shfl_xor_sync(0xffffffffu, send, off);
        }
    }
    return v[0];
}

// Per-column (sum, sum of squares) of the valid rows of one 128-row x 128-column bf16 staging pass
// (two 128-byte-swizzled boxes of 64 columns), read back from shared memory: thread tid takes the
// 8-column chunk tid % 16 of rows 8 (tid / 16) .. + 7 (one conflict-free 16-byte read per row), the two
// row groups of a warp are combined by one shuffle level, and part[w][col][2] gets warp w's partial.
// The statistics are those of the stored bf16 outputs; about 4 instructions per element against ~11
// for the TMEM-register butterfly (FSEL / SHFL: 55 % of the 1x1 forward epilogue's instructions).
template <int COLS>  // 128: two 64-column boxes, 8 rows per thread; 64: one box, 4 rows per thread
__device__ __forceinline__ void pk_tile_stats(const uint8_t *buf, const int *rowm, float *part, int tid) {
    static_assert(COLS == 128 || COLS == 64, "staging pass width");
    constexpr int CG = COLS / 8, RPT = 128 * CG / 256;  // column groups; rows per thread
    const int cg = tid % CG, rg = tid / CG, k = cg >> 3, j = cg & 7;
    int rv[8];
    {
        const int4 m0 = *reinterpret_cast<const int4 *>(rowm + RPT * rg);
        const int4 m1 = RPT == 8 ? *reinterpret_cast<const int4 *>(rowm + RPT * rg + 4) : m0;
        rv[0] = m0.x;
        rv[1] = m0.y;
        rv[2] = m0.z;
        rv[3] = m0.w;
        rv[4] = m1.x;
        rv[5] = m1.y;
        rv[6] = m1.z;
        rv[7] = m1.w;
    }
    // column pairs (2e, 2e + 1) accumulated as packed f32x2 (FADD2 / FFMA2: the same IEEE per-lane
    // rounding as scalar FADD / FFMA, half the instructions of the epilogue's busiest loop)
    uint64_t s2[4] = {0, 0, 0, 0}, q2[4] = {0, 0, 0, 0};
    const uint8_t *base = buf + k * 16384 + (RPT * rg) * 128;
#pragma unroll
    for (int i = 0; i < RPT; ++i) {
        const int r = RPT * rg + i;
        const uint4 w = *reinterpret_cast<const uint4 *>(base + i * 128 + ((j ^ (r & 7)) << 4));
        if (rv[i] < 0) continue;
        const uint32_t u[4] = {w.x, w.y, w.z, w.w};
#pragma unroll
        for (int e = 0; e < 4; ++e) {
            uint64_t x;
            asm("mov.b64 %0, {%1, %2};" : "=l"(x) : "r"(u[e] << 16), "r"(u[e] & 0xffff0000u));
            asm("add.rn.f32x2 %0, %1, %0;" : "+l"(s2[e]) : "l"(x));
            asm("fma.rn.f32x2 %0, %1, %1, %0;" : "+l"(q2[e]) : "l"(x));
        }
    }
    float sm[8], sq[8];
#pragma unroll
    for (int e = 0; e < 4; ++e) {
        asm("mov.b64 {%0, %1}, %2;" : "=f"(sm[2 * e]), "=f"(sm[2 * e + 1]) : "l"(s2[e]));
        asm("mov.b64 {%0, %1}, %2;" : "=f"(sq[2 * e]), "=f"(sq[2 * e + 1]) : "l"(q2[e]));
    }
#pragma unroll
    for (int off = CG; off < 32; off <<= 1)  // the warp's row groups of this column group
#pragma unroll
        for (int c = 0; c < 8; ++c) {
            sm[c] += __shfl_xor_sync(0xffffffffu, sm[c], off);
            sq[c] += __shfl_xor_sync(0xffffffffu, sq[c], off);
        }
    if ((tid & 31) < CG) {
        float4 *o = reinterpret_cast<float4 *>(part + ((tid >> 5) * COLS + cg * 8) * 2);
#pragma unroll
        for (int c = 0; c < 4; ++c) o[c] = make_float4(sm[2 * c], sq[2 * c], sm[2 * c + 1], sq[2 * c + 1]);
    }
}

// Column (sum, sum of squares) of a staged bf16 pass by one 128-thread group (grouped epilogue): rows
// outside the output were staged as zeros, so no row mask; partials part[4 warps][COLS][2].
template <int COLS>
__device__ __forceinline__ void pk_tile_stats_g(const uint8_t *buf, float *part, int gt) {
    static_assert(COLS == 128 || COLS == 64, "staging pass width");
    constexpr int CG = COLS / 8, RPT = 128 * CG / 128;  // column groups; rows per thread
    const int cg = gt % CG, rg = gt / CG, k = cg >> 3, j = cg & 7;
    uint64_t s2[4] = {0, 0, 0, 0}, q2[4] = {0, 0, 0, 0};
    const uint8_t *base = buf + k * 16384 + (RPT * rg) * 128;
#pragma unroll 4
    for (int i = 0; i < RPT; ++i) {
        const int r = RPT * rg + i;
        const uint4 w = *reinterpret_cast<const uint4 *>(base + i * 128 + ((j ^ (r & 7)) << 4));
        const uint32_t u[4] = {w.x, w.y, w.z, w.w};
#pragma unroll
        for (int e = 0; e < 4; ++e) {
            uint64_t x;
            asm("mov.b64 %0, {%1, %2};" : "=l"(x) : "r"(u[e] << 16), "r"(u[e] & 0xffff0000u));
            asm("add.rn.f32x2 %0, %1, %0;" : "+l"(s2[e]) : "l"(x));
            asm("fma.rn.f32x2 %0, %1, %1, %0;" : "+l"(q2[e]) : "l"(x));
        }
    }
    float sm[8], sq[8];
#pragma unroll
    for (int e = 0; e < 4; ++e) {
        asm("mov.b64 {%0, %1}, %2;" : "=f"(sm[2 * e]), "=f"(sm[2 * e + 1]) : "l"(s2[e]));
        asm("mov.b64 {%0, %1}, %2;" : "=f"(sq[2 * e]), "=f"(sq[2 * e + 1]) : "l"(q2[e]));
    }
#pragma unroll
    for (int off = CG; off < 32; off <<= 1)
#pragma unroll
        for (int c = 0; c < 8; ++c) {
            sm[c] += __shfl_xor_sync(0xffffffffu, sm[c], off);
            sq[c] += __shfl_xor_sync(0xffffffffu, sq[c], off);
        }
    if ((gt & 31) < CG) {
        float4 *o = reinterpret_cast<float4 *>(part + ((gt >> 5) * COLS + cg * 8) * 2);
#pragma unroll
        for (int c = 0; c < 4; ++c) o[c] = make_float4(sm[2 * c], sq[2 * c], sm[2 * c + 1], sq[2 * c + 1]);
    }
}

__device__ __forceinline__ void pk_unit(const PkArgs &a, int u, int &tm, int &tn, int &split, int &g) {
    split = u % a.splits;
    const int t = u / a.splits;
    tn = t % a.tiles_n;
    const int r = t / a.tiles_n;
    tm = r % a.tiles_m;
    g = r / a.tiles_m;
}
__device__ __forceinline__ void pk_unit(const PkArgs &a, int u, int &tm, int &tn, int &split) {
    int g;
    pk_unit(a, u, tm, tn, split, g);
}
template <int CL>
__device__ __forceinline__ void pk_unit_cl(const PkArgs &a, int u, int rank, int &tm, int &tn, int &split, int &g) {
    if constexpr (CL == 1) {
        (void)rank;
        pk_unit(a, u, tm, tn, split, g);
    } else {
        split = u % a.splits;
        const int t = u / a.splits;
        tn = t % a.tiles_n;
        const int r = t / a.tiles_n;
        tm = 2 * (r % a.tiles_pm) + rank;
        g = r / a.tiles_pm;
    }
}

// tile row -> output row m (or -1): pixel box rows (FPROP / DGRAD) or m0 + r.
__device__ __forceinline__ int pk_row_m(const PkArgs &a, int tm, int r, int g = 0) {
    if (a.boxed) return conv_box_row(pk_geom(a, g), tm, r);
    const int m = tm * 128 + r;
    return m < a.M ? m : -1;
}

__device__ __forceinline__ uint32_t pk_bf16x2(float a, float b) {
    __nv_bfloat162 h = __floats2bfloat162_rn(a, b);
    return *reinterpret_cast<uint32_t *>(&h);
}

constexpr int kPkThreads = 384;  // 4 control warps + 8 epilogue warps
constexpr int kPkEpi = 256;

// CL = 2: launched as clusters of two CTAs that process M-tile pairs sharing
// (tile_n, split); each CTA loads its own A and half of the common B tile,
// multicast into both CTAs' ring slot; a slot is free once BOTH CTAs' MMAs
// have consumed it (empty barrier count 2, commits multicast to the pair).
template <int KIND, int BN, bool A_MN, bool B_MN, class Epi, int MODE, int CL = 1>
__global__ void __launch_bounds__(kPkThreads, 1)
    gemm_pk_kernel(const __grid_constant__ GemmMaps maps, const __grid_constant__ PkArgs args,
                   const typename Epi::Params ep) {
    using C = PkCfg<KIND, BN, A_MN, B_MN, Epi::kStages, pk_ebuf_bytes<Epi>()>;
    static_assert(CL == 1 || (CL == 2 && MODE != GM_BATCH && MODE != GM_DGRAD && B_MN && BN / C::CH >= 2),
                  "CTA pairs share an MN-major B tile of at least two chunks");
    const int rank = CL == 1 ? 0 : int(ptx::cluster_ctarank());
    const int first = CL == 1 ? int(blockIdx.x) : int(ptx::cluster_id_x());
    const int stride = CL == 1 ? int(gridDim.x) : int(ptx::nclusters_x());
    extern __shared__ __align__(16) uint8_t smem_raw[];
    // 1024-byte alignment by pointer arithmetic on the shared array (keeps the
    // shared address space visible to the compiler: LDS/STS, not generic LD/ST)
    uint8_t *smem = smem_raw + ((1024u - (ptx::smem_u32(smem_raw) & 1023u)) & 1023u);
    uint8_t *sA = smem;
    uint8_t *sB = smem + C::STAGES * C::A_BYTES;
    float *stile = reinterpret_cast<float *>(smem + C::STAGES * C::STAGE_BYTES);
    float *spart = reinterpret_cast<float *>(smem + C::STAGES * C::STAGE_BYTES + C::EPI_BYTES);
    int *rowm = reinterpret_cast<int *>(smem + C::STAGES * C::STAGE_BYTES + C::EPI_BYTES + C::PART_BYTES);
    uint64_t *full = reinterpret_cast<uint64_t *>(rowm + 128);
    uint64_t *empty = full + C::STAGES;
    uint64_t *tfull = empty + C::STAGES;
    uint64_t *tempty = tfull + 2;
    // TMA-staged epilogue operand ring (64-column halves of 128-column passes: BN >= 128)
    constexpr int NES = C::EPI_COLS == 128 ? pk_ebuf_slots<Epi>() : 0;
    // arrivals that free an accumulator: the staged-operand epilogue's two column halves, the direct
    // (register-only) epilogue's eight warps, else one (after a CTA-wide epilogue barrier)
    constexpr int kTemptyArrivals = NES > 0 ? 2 : pk_direct<Epi>::value ? 8 : 1;
    uint64_t *efull = tempty + 2;
    uint64_t *eempty = efull + NES;
    uint32_t *tmem_slot = reinterpret_cast<uint32_t *>(eempty + NES + 1);
    float *spre = reinterpret_cast<float *>(reinterpret_cast<uint8_t *>(rowm) + 512 + 256);  // [2][128][2]
    uint8_t *sones = reinterpret_cast<uint8_t *>(rowm) + 3072;  // 1024-aligned (rowm is)
    // BN statistics of 128-column TMA-store tiles by the tensor core: the column sums and sums of squares
    // of the staged bf16 tile Y are Y^T 1 and diag(Y^T Y), two MMAs into 144 spare TMEM columns
    constexpr bool kMmaStats = Epi::kTmaStore && BN == 128 && KIND == 0;
    constexpr uint32_t kTmemCols = kMmaStats ? 512u : C::TMEM_COLS;
    uint64_t *sbar = eempty + NES;  // the statistics MMAs' commit barrier
    uint8_t *ebuf = smem + C::STAGES * C::STAGE_BYTES;
    static_assert(C::STAGES * 2 + 4 + 2 * NES + 1 <= 30, "barrier area");

    const uint32_t warp = ptx::warp_id();
    if (warp == 0 && ptx::lane_id() == 0) {
        for (int s = 0; s < args.n_seg; ++s) {
            ptx::tma_prefetch_desc(&maps.a[s]);
            ptx::tma_prefetch_desc(&maps.b[s]);
        }
    }
    if (warp == 1 && ptx::lane_id() == 0) {
        for (int s = 0; s < C::STAGES; ++s) {
            ptx::mbar_init(&full[s], 1);
            ptx::mbar_init(&empty[s], CL);
        }
        for (int a = 0; a < 2; ++a) {
            ptx::mbar_init(&tfull[a], 1);
            ptx::mbar_init(&tempty[a], kTemptyArrivals);
        }
        for (int a = 0; a < NES; ++a) {
            ptx::mbar_init(&efull[a], 1);
            ptx::mbar_init(&eempty[a], 4);  // the four TMEM-quarter warps of one column half
        }
        ptx::mbar_init(sbar, 1);
        ptx::fence_barrier_init();
    }
    if (warp == 2) ptx::tmem_alloc<kTmemCols>(tmem_slot);
    if constexpr (kMmaStats) {  // ones [16 rows][128] bf16, K-major 128-byte-swizzled (two 64-column chunks)
        for (int i = threadIdx.x; i < C::ONES_BYTES / 4; i += blockDim.x)
            reinterpret_cast<uint32_t *>(sones)[i] = 0x3F803F80u;
        ptx::fence_proxy_async_smem();
    }
    ptx::tc_fence_before();
    if constexpr (CL == 1)
        __syncthreads();
    else
        ptx::cluster_sync();  // the partner's barriers are initialised before any multicast
    ptx::tc_fence_after();
    const uint32_t tmem_base = *tmem_slot;
    ptx::griddep_wait();
    ptx::griddep_launch();

    if (warp == 0) {
        if (ptx::lane_id() == 0) {
            int it = 0, s = 0, ph = 0;  // ring position: slot s of round ph (it = ph * STAGES + s)
            for (int u = first; u < args.units; u += stride) {
                int tm, tn, sp, g_;
                pk_unit_cl<CL>(args, u, rank, tm, tn, sp, g_);
                const ConvGeom &cg = pk_geom(args, g_);
                const int kbps = args.nph > 1 ? cg.ntap * cg.cpt : args.kb_per_seg;
                const int tot = args.nph > 1 ? kbps * args.n_seg : args.total_iters;
                const int lo = sp * args.iters_per_split, hi = min(tot, lo + args.iters_per_split);
                const int m0 = tm * 128, n0 = tn * BN;
                ConvIter<C, MODE> ci;
                if constexpr (MODE == GM_FPROP || MODE == GM_DGRAD || MODE == GM_WGRAD) ci.init(cg, kbps, lo, tm, m0);
                int seg = lo / args.kb_per_seg, kb = lo - seg * args.kb_per_seg;  // plain / batched modes
                for (int g = lo; g < hi; ++g, ++it) {
                    if (it >= C::STAGES) ptx::mbar_wait(&empty[s], (ph - 1) & 1);
                    ptx::mbar_arrive_expect_tx(&full[s], C::STAGE_BYTES);
                    if constexpr (MODE == GM_PLAIN) {
                        load_operand<C, A_MN, 128>(sA + s * C::A_BYTES, &maps.a[seg], &full[s], m0, kb * C::BK);
                        load_b<C, B_MN, BN, CL>(sB + s * C::B_BYTES, &maps.b[seg], &full[s], n0, kb * C::BK, rank);
                    } else if constexpr (MODE == GM_BATCH) {
                        const int hh = g_ % args.nh, bb = g_ / args.nh, k0 = kb * C::BK;
                        if constexpr (!A_MN) {
                            ptx::tma_load_4d(sA + s * C::A_BYTES, &maps.a[seg], &full[s], k0, m0, hh, bb);
                        } else {
#pragma unroll
                            for (int c = 0; c < 128 / C::CH; ++c)
                                ptx::tma_load_4d(sA + s * C::A_BYTES + c * (C::BK * 128), &maps.a[seg], &full[s],
                                                 m0 + c * C::CH, k0, hh, bb);
                        }
                        if constexpr (!B_MN) {
                            ptx::tma_load_4d(sB + s * C::B_BYTES, &maps.b[seg], &full[s], k0, n0, hh, bb);
                        } else {
#pragma unroll
                            for (int c = 0; c < BN / C::CH; ++c)
                                ptx::tma_load_4d(sB + s * C::B_BYTES + c * (C::BK * 128), &maps.b[seg], &full[s],
                                                 n0 + c * C::CH, k0, hh, bb);
                        }
                    } else {
                        ci.template load<B_MN, BN, CL>(sA + s * C::A_BYTES, sB + s * C::B_BYTES, maps, cg, &full[s],
                                                       n0, rank);
                        ci.next(cg);
                    }
                    if (++kb == args.kb_per_seg) {
                        kb = 0;
                        ++seg;
                    }
                    if (++s == C::STAGES) {
                        s = 0;
                        ++ph;
                    }
                }
            }
        }
    } else if (warp == 1) {
        if (ptx::lane_id() == 0) {
            int s = 0, ph = 0, j = 0;
            for (int u = first; u < args.units; u += stride, ++j) {
                int tm, tn, sp, g_;
                pk_unit_cl<CL>(args, u, rank, tm, tn, sp, g_);
                const int tot = args.nph > 1 ? pk_geom(args, g_).ntap * pk_geom(args, g_).cpt * args.n_seg
                                             : args.total_iters;
                const int lo = sp * args.iters_per_split, hi = min(tot, lo + args.iters_per_split);
                const int acc = j & 1;
                if (j >= 2) ptx::mbar_wait(&tempty[acc], ((j >> 1) - 1) & 1);
                ptx::tc_fence_after();
                const uint32_t d = tmem_base + uint32_t(acc * BN);
                for (int g = lo; g < hi; ++g) {
                    ptx::mbar_wait(&full[s], ph & 1);
                    ptx::tc_fence_after();
                    const uint32_t a_base = ptx::smem_u32(sA + s * C::A_BYTES);
                    const uint32_t b_base = ptx::smem_u32(sB + s * C::B_BYTES);
#pragma unroll
                    for (int k = 0; k < C::BK / C::UMMA_K; ++k)
                        ptx::umma<KIND>(d, operand_desc<C, A_MN>(a_base, k), operand_desc<C, B_MN>(b_base, k), C::IDESC,
                                        (g > lo || k > 0) ? 1u : 0u);
                    if constexpr (CL == 1)
                        ptx::umma_commit(&empty[s]);
                    else
                        ptx::umma_commit_mc(&empty[s], 3);
                    if (++s == C::STAGES) {
                        s = 0;
                        ++ph;
                    }
                }
                ptx::umma_commit(&tfull[acc]);
            }
        }
    } else if (warp == 3) {
        // epilogue operand producer (kTmaAdd): per unit, per 64-column chunk, one TMA box of the
        // residual gradient (and one of its mask) into the next ring slot, as early as the ring allows
        if constexpr (NES > 0) {
            if (ptx::lane_id() == 0) {
                constexpr int NCH = BN / 64;
                const uint32_t bytes = args.tma_add == 2 ? 32768u : 16384u;
                int seq = 0;
                for (int u = first; u < args.units; u += stride) {
                    int tm, tn, sp, g_;
                    pk_unit_cl<CL>(args, u, rank, tm, tn, sp, g_);
                    int w0 = 0, h0 = 0, b0 = 0;
                    if (args.boxed) conv_box_origin(args.cv, tm, w0, h0, b0);
#pragma unroll 1
                    for (int k = 0; k < NCH; ++k, ++seq) {
                        const int slot = seq % NES;
                        if (seq >= NES) ptx::mbar_wait(&eempty[slot], ((seq / NES) - 1) & 1);
                        ptx::mbar_arrive_expect_tx(&efull[slot], bytes);
                        uint8_t *dst = ebuf + slot * 32768;
                        const int col = tn * BN + k * 64;
#pragma unroll 1
                        for (int o = 0; o < args.tma_add; ++o) {
                            if (args.boxed)
                                ptx::tma_load_4d(dst + o * 16384, &maps.e[o], &efull[slot], col, w0, h0, b0);
                            else
                                ptx::tma_load_2d(dst + o * 16384, &maps.e[o], &efull[slot], col, tm * 128);
                        }
                    }
                }
            }
        }
    } else if (warp >= 4) {
        const int tid = threadIdx.x - 128;  // 0..255
        const int q = warp & 3;             // TMEM lane quarter this warp may access
        const int half = (warp - 4) >> 2;   // column half of each staging pass
        const int row = q * 32 + ptx::lane_id();
        constexpr int HC = C::EPI_COLS / 2;
        bool grouped_run = false;
        if constexpr (Epi::kTmaStore && NES == 0) {
            if (args.grouped) {  // PkArgs::grouped: group `half` takes the units of accumulator `half`
                const int gt = row, grp = half, gbar = 3 + grp;
                uint8_t *buf = smem + C::STAGES * C::STAGE_BYTES + grp * (C::EPI_COLS * 256);
                float *gpart = spart + grp * (4 * C::EPI_COLS * 2);
                float *gpre = grp == 0 ? spre : reinterpret_cast<float *>(sones);  // [2 passes][128][2]
                const int nsl = 2 * int(gridDim.x), sl = 2 * int(blockIdx.x) + grp;
                const bool stats = Epi::has_stats(ep);
                Epi::gstats_init(ep, args.N, gt, nsl, sl);
                int j = 0;
                for (int u = first; u < args.units; u += stride, ++j) {
                    if ((j & 1) != grp) continue;
                    int tm, tn, sp, g;
                    pk_unit_cl<CL>(args, u, rank, tm, tn, sp, g);
                    if (CL > 1 && tm >= args.tiles_m) {  // phantom tile: release the accumulator unread
                        if (gt == 0) {
                            ptx::mbar_wait(&tfull[grp], (j >> 1) & 1);
                            ptx::mbar_arrive(&tempty[grp]);
                        }
                        continue;
                    }
#pragma unroll
                    for (int h = 0; h < BN / C::EPI_COLS; ++h) {
                        const int c0 = tn * BN + h * C::EPI_COLS;
                        Epi::gstats_pre(ep, c0, min(C::EPI_COLS, args.N - c0), gt, gpre + h * 256, nsl, sl);
                    }
                    const bool live = pk_row_m(args, tm, row, g) >= 0;
                    ptx::mbar_wait(&tfull[grp], (j >> 1) & 1);
                    ptx::tc_fence_after();
                    const uint32_t taddr = tmem_base + (uint32_t(q * 32) << 16) + uint32_t(grp * BN);
#pragma unroll 1
                    for (int h = 0; h < BN / C::EPI_COLS; ++h) {
#pragma unroll 1
                        for (int c = 0; c < C::EPI_COLS; c += 32) {
                            float v[32];
                            ptx::tmem_ld32(taddr + h * C::EPI_COLS + c, v);
                            uint8_t *rp = buf + (c >> 6) * 16384 + row * 128;
                            const int u0 = (c & 63) >> 3;
#pragma unroll
                            for (int i = 0; i < 4; ++i) {
                                uint4 w;
                                w.x = pk_bf16x2(v[8 * i], v[8 * i + 1]);
                                w.y = pk_bf16x2(v[8 * i + 2], v[8 * i + 3]);
                                w.z = pk_bf16x2(v[8 * i + 4], v[8 * i + 5]);
                                w.w = pk_bf16x2(v[8 * i + 6], v[8 * i + 7]);
                                if (!live) w = make_uint4(0u, 0u, 0u, 0u);  // never stored; zero for the statistics
                                *reinterpret_cast<uint4 *>(rp + (((u0 + i) ^ (row & 7)) << 4)) = w;
                            }
                        }
                        ptx::fence_proxy_async_smem();
                        if (h == BN / C::EPI_COLS - 1) ptx::tc_fence_before();
                        pk_bar(gbar, 128);
                        if (h == BN / C::EPI_COLS - 1 && gt == 0) ptx::mbar_arrive(&tempty[grp]);
                        const int col0 = tn * BN + h * C::EPI_COLS;
                        if (gt == 0) {
#pragma unroll 1
                            for (int k = 0; k < C::EPI_COLS / 64; ++k) {
                                const int col = col0 + k * 64;
                                if (col >= args.N) break;
                                const uint8_t *src = buf + k * 16384;
                                if (args.boxed) {
                                    int w0, h0, b0;
                                    conv_box_origin(args.cv, tm, w0, h0, b0);
                                    ptx::tma_store_4d(&maps.o, src, col, w0, h0, b0);
                                } else {
                                    ptx::tma_store_2d(&maps.o, src, col, tm * 128);
                                }
                            }
                            ptx::bulk_commit();
                        }
                        if (stats) {
                            pk_tile_stats_g<C::EPI_COLS>(buf, gpart, gt);
                            pk_bar(gbar, 128);
                            Epi::gstats_add(ep, gpart, C::EPI_COLS, col0, min(C::EPI_COLS, args.N - col0), gt,
                                            gpre + h * 256, nsl, sl);
                        }
                        if (gt == 0) ptx::bulk_wait_read0();  // the buffer is rewritten by the next pass
                        pk_bar(gbar, 128);                    // (and gpart by the next statistics)
                    }
                }
                if (gt == 0) ptx::bulk_wait0();  // TMA stores complete before the CTA exits
                grouped_run = true;
            }
        }
        if (!grouped_run) {
        if (args.splits == 1) {
            Epi::template col_stats_init<kPkEpi>(ep, args.N, C::EPI_COLS, tid);
            pk_bar(1, kPkEpi);
        }
        // bf16 staging of the TMA store (aliases stile): two buffers of one pass (EPI_COLS columns) each,
        // alternating per pass; a buffer is rewritten only after its previous store group was read
        uint8_t *stage = smem + C::STAGES * C::STAGE_BYTES;
        static_assert(!Epi::kTmaStore || 2 * C::EPI_COLS * 256 <= C::STILE_BYTES, "TMA staging exceeds the shared tile");
        int pc = 0;  // TMA passes issued by this CTA
        int j = 0;
        for (int u = first; u < args.units; u += stride, ++j) {
            int tm, tn, sp, g;
            pk_unit_cl<CL>(args, u, rank, tm, tn, sp, g);
            if (CL > 1 && tm >= args.tiles_m) {  // phantom tile: release the accumulator unread
                if (tid == 0) {
                    ptx::mbar_wait(&tfull[j & 1], (j >> 1) & 1);
                    for (int k = 0; k < kTemptyArrivals; ++k) ptx::mbar_arrive(&tempty[j & 1]);
                }
                continue;
            }
            const int64_t out_off = MODE == GM_BATCH ? (g / args.nh) * args.out_bs + (g % args.nh) * args.out_hs : 0;
            const int acc = j & 1;
            const bool split = args.splits > 1;
            const bool tma = Epi::kTmaStore && args.tma_out && !split;
            static_assert(BN / C::EPI_COLS <= 2 && C::EPI_COLS <= 128, "statistics prefetch slots");
            if (!split) {  // the running statistics of the unit's columns, copied asynchronously (no register
                           // waits on them; col_stats waits for the thread's own copies)
#pragma unroll
                for (int h = 0; h < BN / C::EPI_COLS; ++h) {
                    const int c0 = tn * BN + h * C::EPI_COLS;
                    Epi::col_stats_pre(ep, c0, min(C::EPI_COLS, args.N - c0), tid, spre + h * 256);
                }
            }
            if (tid < 128) {  // the previous unit's last barrier protects rowm / stile
                const int m = pk_row_m(args, tm, tid, g);
                rowm[tid] = m;
                if (!split) Epi::prefetch_row(ep, m, tn * BN, min(BN, args.N - tn * BN), out_off);
            }
            if constexpr (NES > 0) {  // direct epilogue on TMA-staged residual / mask rows (no split)
                const int row_m = pk_row_m(args, tm, row, g);
                typename Epi::DirectPre dp;
                ptx::mbar_wait(&tfull[acc], (j >> 1) & 1);
                ptx::tc_fence_after();
                const uint32_t taddr = tmem_base + (uint32_t(q * 32) << 16) + uint32_t(acc * BN);
#pragma unroll 1
                for (int h = 0; h < BN / C::EPI_COLS; ++h) {
                    const int seq = j * (BN / 64) + 2 * h + half, slot = seq % NES;
                    uint8_t *sl = ebuf + slot * 32768;
                    const int mask = ep.mul ? 3 : args.tma_add == 2 ? (ep.add_mask.hi ? 1 : 2) : 0;
                    ptx::mbar_wait(&efull[slot], (seq / NES) & 1);
                    Epi::smem_load(sl, row, mask == 1 || mask == 2, dp);
                    const int col = tn * BN + h * C::EPI_COLS + half * HC;
                    if (args.tma_out) {  // output through the slot: bf16 over the residual, one TMA store
#pragma unroll
                        for (int qq = 0; qq < HC / 16; ++qq) {
                            float v[16];
                            ptx::tmem_ld16(taddr + h * C::EPI_COLS + half * HC + 16 * qq, v);
                            Epi::smem_store(sl, row, qq, mask, dp, v);  // (mask: 0 none, 1 residual, 2 sum)
                        }
                        ptx::fence_proxy_async_smem();
                        pk_bar(3 + half, 128);  // the half's four warps wrote their rows
                        if (q == 0 && ptx::lane_id() == 0) {
                            if (args.boxed) {
                                int w0, h0, b0;
                                conv_box_origin(args.cv, tm, w0, h0, b0);
                                ptx::tma_store_4d(&maps.o, sl, col, w0, h0, b0);
                            } else {
                                ptx::tma_store_2d(&maps.o, sl, col, tm * 128);
                            }
                            ptx::bulk_commit();
                            ptx::bulk_wait_read0();  // the slot is reusable once the store has read it
                        }
                        __syncwarp();
                        if (ptx::lane_id() == 0) ptx::mbar_arrive(&eempty[slot]);
                    } else {
                        __syncwarp();
                        if (ptx::lane_id() == 0) ptx::mbar_arrive(&eempty[slot]);
#pragma unroll
                        for (int qq = 0; qq < HC / 16; ++qq) {
                            float v[16];
                            ptx::tmem_ld16(taddr + h * C::EPI_COLS + half * HC + 16 * qq, v);
                            Epi::direct_store(ep, row_m, col, qq, out_off, dp, v);
                        }
                    }
                }
                // each column half frees the accumulator for itself (no CTA-wide barrier per unit: the halves
                // only meet in the operand ring's order)
                ptx::tc_fence_before();
                pk_bar(3 + half, 128);
                if (q == 0 && ptx::lane_id() == 0) ptx::mbar_arrive(&tempty[acc]);
                continue;
            } else if constexpr (pk_direct<Epi>::value) {  // the only epilogue of this instantiation (no split)
                const int row_m = pk_row_m(args, tm, row, g);
                typename Epi::DirectPre dp;
                Epi::template direct_load<HC>(ep, row_m, tn * BN + half * HC, out_off, dp);  // before the accumulator
                ptx::mbar_wait(&tfull[acc], (j >> 1) & 1);
                ptx::tc_fence_after();
                const uint32_t taddr = tmem_base + (uint32_t(q * 32) << 16) + uint32_t(acc * BN);
#pragma unroll 1
                for (int h = 0; h < BN / C::EPI_COLS; ++h) {
                    const int col = tn * BN + h * C::EPI_COLS + half * HC;
                    if (h > 0) Epi::template direct_load<HC>(ep, row_m, col, out_off, dp);
#pragma unroll
                    for (int qq = 0; qq < HC / 16; ++qq) {
                        float v[16];
                        ptx::tmem_ld16(taddr + h * C::EPI_COLS + half * HC + 16 * qq, v);
                        Epi::direct_store(ep, row_m, col, qq, out_off, dp, v);
                    }
                }
                // every warp frees the accumulator for itself: no CTA-wide barrier per unit (nothing shared)
                ptx::tc_fence_before();
                __syncwarp();
                if (ptx::lane_id() == 0) ptx::mbar_arrive(&tempty[acc]);
                continue;
            } else {
            ptx::mbar_wait(&tfull[acc], (j >> 1) & 1);
            ptx::tc_fence_after();
            const uint32_t taddr = tmem_base + (uint32_t(q * 32) << 16) + uint32_t(acc * BN);
            if constexpr (Epi::kTmaStore) {
                if (tma) {
                    const int row_m = pk_row_m(args, tm, row, g);
                    const bool stats = Epi::has_stats(ep);
#pragma unroll 1
                    for (int h = 0; h < BN / C::EPI_COLS; ++h, ++pc) {
                        uint8_t *buf = stage + (pc & 1) * (C::EPI_COLS * 256);
#pragma unroll 1
                        for (int c = half * HC; c < (half + 1) * HC; c += 32) {
                            const int uc = h * C::EPI_COLS + c;  // column within the unit
                            float v[32];
                            ptx::tmem_ld32(taddr + uc, v);
                            uint8_t *rp = buf + (c >> 6) * 16384 + row * 128;
                            const int u0 = (c & 63) >> 3;
#pragma unroll
                            for (int i = 0; i < 4; ++i) {
                                uint4 w;
                                w.x = pk_bf16x2(v[8 * i], v[8 * i + 1]);
                                w.y = pk_bf16x2(v[8 * i + 2], v[8 * i + 3]);
                                w.z = pk_bf16x2(v[8 * i + 4], v[8 * i + 5]);
                                w.w = pk_bf16x2(v[8 * i + 6], v[8 * i + 7]);
                                // rows outside the output (never stored) are zero for the statistics MMAs
                                if (kMmaStats && args.mma_stats && row_m < 0) w = make_uint4(0u, 0u, 0u, 0u);
                                *reinterpret_cast<uint4 *>(rp + (((u0 + i) ^ (row & 7)) << 4)) = w;
                            }
                        }
                        ptx::fence_proxy_async_smem();  // staging writes -> async proxy (TMA store / MMA)
                        if (h == BN / C::EPI_COLS - 1) ptx::tc_fence_before();
                        pk_bar(1, kPkEpi);
                        if (h == BN / C::EPI_COLS - 1 && tid == 0) ptx::mbar_arrive(&tempty[acc]);
                        const int col0 = tn * BN + h * C::EPI_COLS;
                        if (tid == 0) {
#pragma unroll 1
                            for (int k = 0; k < C::EPI_COLS / 64; ++k) {
                                const int col = col0 + k * 64;
                                if (col >= args.N) break;
                                const uint8_t *src = buf + k * 16384;
                                if (args.boxed) {
                                    int w0, h0, b0;
                                    conv_box_origin(args.cv, tm, w0, h0, b0);
                                    ptx::tma_store_4d(&maps.o, src, col, w0, h0, b0);
                                } else {
                                    ptx::tma_store_2d(&maps.o, src, col, tm * 128);
                                }
                            }
                            ptx::bulk_commit();
                            ptx::bulk_wait_read1();  // the other buffer (previous pass) is free again
                        }
                        if (stats) {
                            if (kMmaStats && args.mma_stats) {  // diag(Y^T Y) and Y^T 1 of the staged tile
                                if (tid == 0) {
                                    ptx::tc_fence_after();
                                    const uint32_t yb = ptx::smem_u32(buf), ob = ptx::smem_u32(sones);
                                    constexpr uint32_t idG = ptx::instr_desc(1, true, true, 128, 128);
                                    constexpr uint32_t idS = ptx::instr_desc(1, true, false, 128, 16);
#pragma unroll
                                    for (int k = 0; k < 8; ++k) {  // 16 rows per step
                                        const uint64_t ya = ptx::smem_desc_sw128(yb + k * 2048, 16384, 1024);
                                        ptx::umma<0>(tmem_base + 256, ya, ya, idG, k > 0 ? 1u : 0u);
                                        ptx::umma<0>(tmem_base + 384, ya,
                                                     ptx::smem_desc_sw128(ob + (k >> 2) * 2048 + (k & 3) * 32, 16, 1024),
                                                     idS, k > 0 ? 1u : 0u);
                                    }
                                    ptx::umma_commit(sbar);
                                }
                                if (warp < 8) {  // warps 4-7: TMEM lanes = the pass's 128 columns
                                    ptx::mbar_wait(sbar, uint32_t(pc) & 1u);
                                    ptx::tc_fence_after();
                                    const uint32_t ta = tmem_base + (uint32_t(q * 32) << 16);
                                    float v[32], cs[1];
                                    ptx::tmem_ld32(ta + 256 + q * 32, v);
                                    ptx::tmem_ld1(ta + 384, cs);
                                    float sq = 0.f;
#pragma unroll
                                    for (int k = 0; k < 32; ++k) sq = ptx::lane_id() == k ? v[k] : sq;
                                    Epi::col_stats_value(ep, col0, min(C::EPI_COLS, args.N - col0), tid, cs[0], sq,
                                                         spre + h * 256);
                                    ptx::tc_fence_before();
                                }
                            } else {  // from the stored bf16 tile (staging read-back)
                                pk_tile_stats<C::EPI_COLS>(buf, rowm, spart, tid);
                                pk_bar(1, kPkEpi);
                                Epi::col_stats8(ep, spart, C::EPI_COLS, col0, min(C::EPI_COLS, args.N - col0), tid,
                                                spre + h * 256);
                            }
                        }
                        pk_bar(1, kPkEpi);  // spart / staging reused by the next pass
                    }
                    continue;
                }
            }
#pragma unroll 1
            for (int h = 0; h < BN / C::EPI_COLS; ++h) {
                const int row_m = pk_row_m(args, tm, row, g);  // own computation: rowm is not yet synced
#pragma unroll 1
                for (int c = half * HC; c < (half + 1) * HC; c += 32) {
                    float v[32];
                    ptx::tmem_ld32(taddr + h * C::EPI_COLS + c, v);
                    // epilogue drain hook (whole warp, lockstep): may fold extra operands into the
                    // row and reduce per-column statistics into spart[q][c + lane][0..2]
                    Epi::drain(ep, split, row_m, tn * BN + h * C::EPI_COLS + c, v, stile + row * C::LDS + c,
                               spart + (q * C::EPI_COLS + c + ptx::lane_id()) * 3);
                }
                if (h == BN / C::EPI_COLS - 1) ptx::tc_fence_before();
                pk_bar(1, kPkEpi);
                if (h == BN / C::EPI_COLS - 1 && tid == 0) ptx::mbar_arrive(&tempty[acc]);  // accumulator free
                const int col0 = tn * BN + h * C::EPI_COLS;
                if (split) {
                    float *dst = args.ws + ((size_t(tm) * args.tiles_n + tn) * args.splits + sp) * 128 * BN +
                                 h * C::EPI_COLS;
                    constexpr int C4 = C::EPI_COLS / 4;
                    for (int e = tid; e < 128 * C4; e += kPkEpi) {
                        const int r = e / C4, cc = (e % C4) * 4;
                        *reinterpret_cast<float4 *>(dst + size_t(r) * BN + cc) =
                            *reinterpret_cast<const float4 *>(stile + r * C::LDS + cc);
                    }
                } else {
                    const int ncols = min(C::EPI_COLS, args.N - col0);
                    if (ncols == C::EPI_COLS)
                        Epi::template run<kPkEpi, C::EPI_COLS>(ep, stile, C::LDS, rowm, 128, col0, ncols, tm, args.N,
                                                               tid, out_off);
                    else
                        Epi::template run<kPkEpi, 0, true>(ep, stile, C::LDS, rowm, 128, col0, ncols, tm, args.N, tid,
                                                           out_off);
                    Epi::template col_stats<kPkEpi>(ep, spart, C::EPI_COLS, col0, ncols, tm, tid, spre + h * 256);
                }
                pk_bar(1, kPkEpi);  // shared tile reused by the next pass / unit
            }
            if (!split) Epi::template done<kPkEpi>(ep, tid, unsigned(args.tiles_m * args.tiles_n));
            }
        }
        if constexpr (Epi::kTmaStore)
            if (tid == 0) ptx::bulk_wait0();  // TMA stores complete before the CTA exits
        if constexpr (NES > 0)
            if (q == 0 && ptx::lane_id() == 0) ptx::bulk_wait0();  // the slot stores of both halves
        }
    }
    ptx::tc_fence_before();
    if constexpr (CL == 1)
        __syncthreads();
    else
        ptx::cluster_sync();  // the partner's last multicast commits have landed
    if (warp == 2) ptx::tmem_dealloc<kTmemCols>(tmem_base);
}

// Split-K tail: per (tile, row chunk of RC rows, column chunk of CC columns),
// sum the split partials in split order into shared memory and run the
// epilogue on that sub-tile.  256 threads.
template <int BN, class Epi, int RC, int CC>
__global__ void __launch_bounds__(256) pk_reduce_kernel(const __grid_constant__ PkArgs args,
                                                        const typename Epi::Params ep) {
    ptx::griddep_wait();
    ptx::griddep_launch();
    __shared__ __align__(16) float st[RC * (CC + 4)];
    __shared__ int rowm[RC];
    const int tile = blockIdx.x;
    const int tm = tile / args.tiles_n, tn = tile % args.tiles_n;
    const int row0 = blockIdx.y * RC, c0 = blockIdx.z * CC;
    for (int r = threadIdx.x; r < RC; r += 256) rowm[r] = pk_row_m(args, tm, row0 + r);
    const float *base = args.ws + size_t(tile) * args.splits * 128 * BN;
    constexpr int C4 = CC / 4;
    for (int e = threadIdx.x; e < RC * C4; e += 256) {
        const int r = e / C4, c = (e % C4) * 4;
        const float *p = base + size_t(row0 + r) * BN + c0 + c;
        float4 acc = __ldcg(reinterpret_cast<const float4 *>(p));
#pragma unroll 8
        for (int z = 1; z < args.splits; ++z) {
            const float4 t = __ldcg(reinterpret_cast<const float4 *>(p + size_t(z) * 128 * BN));
            acc.x += t.x;
            acc.y += t.y;
            acc.z += t.z;
            acc.w += t.w;
        }
        *reinterpret_cast<float4 *>(st + r * (CC + 4) + c) = acc;
    }
    __syncthreads();
    const int col0 = tn * BN + c0;
    // statistics slot of this row chunk: tm * (128 / RC) + chunk (the caller sizes ep.tiles accordingly)
    Epi::template run_with_stats<256>(ep, st, CC + 4, rowm, RC, col0, min(CC, args.N - col0),
                                      tm * (128 / RC) + int(blockIdx.y), args.N, threadIdx.x, 0);
    Epi::template done<256>(ep, threadIdx.x, gridDim.x * gridDim.y * gridDim.z);
}

// ---------------------------------------------------------------- host side
// CTA pairs are opt-in (CDP_PK_PAIRS=1): measured on B200 they are 1-4% slower than single
// CTAs on ResNet-18/50 and ViT-B/16 (the operand fetch is not what bounds these GEMMs).
inline bool pk_pairs_enabled() {
    static const bool on = [] {
        const char *e = std::getenv("CDP_PK_PAIRS");
        return e && e[0] == '1';
    }();
    return on;
}

// Split-K: at least this many k-blocks per split (CDP_SPLIT_MIN_KB, default 16: 0.6 % faster on
// ResNet-18 than 4; fp32 mode caps its units at one 3xTF32 segment regardless).
inline int split_min_kb() {
    static const int v = [] {
        const char *e = std::getenv("CDP_SPLIT_MIN_KB");
        const int k = e ? std::atoi(e) : 0;
        return k > 0 ? k : 16;
    }();
    return v;
}

// Grid choice and launch of gemm_pk_kernel for prepared args (units = tiles x splits).
template <int KIND, int BN, bool A_MN, bool B_MN, class Epi, int MODE>
struct PkLaunch {
    using C = PkCfg<KIND, BN, A_MN, B_MN, Epi::kStages, pk_ebuf_bytes<Epi>()>;
    static constexpr bool kPairable = MODE != GM_BATCH && MODE != GM_DGRAD && B_MN && BN / C::CH >= 2;

    // Decide pairing (M tiles >= 2, pairable shape), fix up a.tiles_pm / a.units; returns the grid.
    static int prepare(PkArgs &a, int sms, bool &paired) {
        paired = false;
        if constexpr (kPairable) {
            if (pk_pairs_enabled() && a.tiles_m >= 2) {
                paired = true;
                a.tiles_pm = (a.tiles_m + 1) / 2;
                a.units = a.tiles_pm * a.tiles_n * (a.nbatch > 0 ? a.nbatch : 1) * a.splits;
                static int max_pairs = 0;
                if (!max_pairs) {
                    set_attr();
                    max_pairs = std::max(1, max_active_clusters(gemm_pk_kernel<KIND, BN, A_MN, B_MN, Epi, MODE, 2>,
                                                                kPkThreads, C::SMEM, 2));
                }
                return 2 * std::min(a.units, max_pairs);
            }
        }
        return std::min(a.units, sms);
    }
    // TMA-store epilogue for plain bf16 outputs of non-split units (CDP_PK_TMA_STORE=0 disables).
    static void setup_tma_out(GemmMaps &maps, PkArgs &a, const typename Epi::Params &ep) {
        a.tma_out = 0;
        if constexpr (Epi::kTmaStore) {
            static const bool on = [] {
                const char *e = std::getenv("CDP_PK_TMA_STORE");
                return !(e && e[0] == '0');
            }();
            if (!on || a.splits > 1 || MODE == GM_BATCH || MODE == GM_WGRAD || a.N < 64 || !Epi::tma_eligible(ep))
                return;
            const uint64_t rs = uint64_t(ep.ld) * 2;
            if (MODE == GM_PLAIN) {
                maps.o = make_tmap_2d(ep.out, ElemType::BF16, uint64_t(a.N), uint64_t(a.M), rs, 64, 128);
            } else {
                const ConvGeom &g = a.cv;
                if (g.omul != 1 || g.oH != g.Ho || g.oW != g.Wo) return;  // sub-pixel phase outputs
                const uint64_t dims[4] = {uint64_t(a.N), uint64_t(g.Wo), uint64_t(g.Ho), uint64_t(g.Bn)};
                const uint64_t str[3] = {rs, rs * g.Wo, rs * g.Wo * g.Ho};
                const uint32_t box[4] = {64, uint32_t(g.bw), uint32_t(g.bh), uint32_t(g.bn)};
                const uint32_t es[4] = {1, 1, 1, 1};
                maps.o = make_tmap_4d(ep.out, ElemType::BF16, dims, str, box, es, CU_TENSOR_MAP_SWIZZLE_128B);
            }
            a.tma_out = 1;
            static const bool mma_on = [] {
                const char *e = std::getenv("CDP_MMA_STATS");
                return e && e[0] == '1';
            }();
            a.mma_stats = (mma_on && BN == 128 && KIND == 0) ? 1 : 0;
            static const bool grouped_on = [] {
                const char *e = std::getenv("CDP_PK_GROUPED");
                return !(e && e[0] == '0');
            }();
            a.grouped = (grouped_on && !a.mma_stats) ? 1 : 0;
        }
    }
    // TMA-staged epilogue operands (Epi::kTmaAdd): maps of the residual gradient and its mask with the
    // output's tile geometry (boxes of 64 columns x the 128 tile rows).
    static void setup_tma_add(GemmMaps &maps, PkArgs &a, const typename Epi::Params &ep) {
        a.tma_add = 0;
        if constexpr (pk_tma_add<Epi>::value) {
            CDP_REQUIRE(a.splits == 1 && MODE != GM_BATCH && MODE != GM_WGRAD && BN >= 128 && a.N % BN == 0,
                        "TMA-staged epilogue operands: unsplit plain / stride-1 conv tiles of 128 or 256 columns");
            const uint64_t rs = uint64_t(ep.ld) * 2;
            CDP_REQUIRE(!(ep.add_mask.hi && ep.out_mask.hi), "one mask per residual-add epilogue");
            const void *src[2] = {ep.add ? ep.add : ep.mul, ep.add_mask.hi ? ep.add_mask.hi : ep.out_mask.hi};
            const int n = src[1] ? 2 : 1;
            for (int o = 0; o < n; ++o) {
                if (MODE == GM_PLAIN) {
                    maps.e[o] = make_tmap_2d(src[o], ElemType::BF16, uint64_t(a.N), uint64_t(a.M), rs, 64, 128);
                } else {
                    const ConvGeom &g = a.cv;
                    CDP_REQUIRE(g.omul == 1 && g.oH == g.Ho && g.oW == g.Wo, "TMA-staged operands: stride-1 tiles");
                    const uint64_t dims[4] = {uint64_t(a.N), uint64_t(g.Wo), uint64_t(g.Ho), uint64_t(g.Bn)};
                    const uint64_t str[3] = {rs, rs * g.Wo, rs * g.Wo * g.Ho};
                    const uint32_t box[4] = {64, uint32_t(g.bw), uint32_t(g.bh), uint32_t(g.bn)};
                    const uint32_t es[4] = {1, 1, 1, 1};
                    maps.e[o] = make_tmap_4d(src[o], ElemType::BF16, dims, str, box, es, CU_TENSOR_MAP_SWIZZLE_128B);
                }
            }
            a.tma_add = n;
            // output boxes stored from the slots (CDP_TMA_ADD_STORE=0: direct 16-byte stores)
            static const bool st_on = [] {
                const char *e = std::getenv("CDP_TMA_ADD_STORE");
                return !(e && e[0] == '0');
            }();
            a.tma_out = 0;
            if (st_on && (reinterpret_cast<uintptr_t>(ep.out) & 15) == 0) {
                if (MODE == GM_PLAIN) {
                    maps.o = make_tmap_2d(ep.out, ElemType::BF16, uint64_t(a.N), uint64_t(a.M), rs, 64, 128);
                } else {
                    const ConvGeom &g = a.cv;
                    const uint64_t dims[4] = {uint64_t(a.N), uint64_t(g.Wo), uint64_t(g.Ho), uint64_t(g.Bn)};
                    const uint64_t str[3] = {rs, rs * g.Wo, rs * g.Wo * g.Ho};
                    const uint32_t box[4] = {64, uint32_t(g.bw), uint32_t(g.bh), uint32_t(g.bn)};
                    const uint32_t es[4] = {1, 1, 1, 1};
                    maps.o = make_tmap_4d(ep.out, ElemType::BF16, dims, str, box, es, CU_TENSOR_MAP_SWIZZLE_128B);
                }
                a.tma_out = 1;
            }
        }
    }
    static void set_attr() {
        static bool done = false;
        if (done) return;
        CDP_CUDA(cudaFuncSetAttribute(gemm_pk_kernel<KIND, BN, A_MN, B_MN, Epi, MODE, 1>,
                                      cudaFuncAttributeMaxDynamicSharedMemorySize, C::SMEM));
        if constexpr (kPairable)
            CDP_CUDA(cudaFuncSetAttribute(gemm_pk_kernel<KIND, BN, A_MN, B_MN, Epi, MODE, 2>,
                                          cudaFuncAttributeMaxDynamicSharedMemorySize, C::SMEM));
        done = true;
    }
    static void launch(const GemmMaps &maps, const PkArgs &a, const typename Epi::Params &ep, cudaStream_t s, int grid,
                       bool paired) {
        set_attr();
        if constexpr (kPairable) {
            if (paired) {
                launch_pdl_cluster(gemm_pk_kernel<KIND, BN, A_MN, B_MN, Epi, MODE, 2>, dim3(grid), dim3(kPkThreads),
                                   C::SMEM, s, 2, maps, a, ep);
                return;
            }
        }
        launch_pdl(gemm_pk_kernel<KIND, BN, A_MN, B_MN, Epi, MODE, 1>, dim3(grid), dim3(kPkThreads), C::SMEM, s, maps,
                   a, ep);
    }
};

}  // namespace cdp
