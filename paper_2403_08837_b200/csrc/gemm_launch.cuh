// Host-side launch helpers for gemm_tc_kernel.
#pragma once
#include <algorithm>
#include <cstring>

#include "gemm.cuh"
#include "host.h"

namespace cdp {

// Operand view: element type, majorness, extents, row stride.
//  K-major : element (mn, k) at base[mn * ld + k]
//  MN-major: element (mn, k) at base[k * ld + mn]
struct Operand {
    const void *ptr = nullptr;
    bool mn_major = false;
    uint64_t mn = 0, k = 0;   // logical extents
    uint64_t ld = 0;          // leading dimension in elements
};

template <int KIND>
inline CUtensorMap operand_map(const Operand &o, int tile_rows) {
    constexpr int ELEM = KIND == 0 ? 2 : 4;
    constexpr uint32_t CH = 128 / ELEM;
    const ElemType t = KIND == 0 ? ElemType::BF16 : ElemType::F32;
    if (!o.mn_major) return make_tmap_2d(o.ptr, t, o.k, o.mn, o.ld * ELEM, CH, uint32_t(tile_rows));
    return make_tmap_2d(o.ptr, t, o.mn, o.k, o.ld * ELEM, CH, CH,
                        KIND == 0 ? CU_TENSOR_MAP_SWIZZLE_128B : CU_TENSOR_MAP_SWIZZLE_128B_ATOM_32B);
}

struct GemmPlan {
    GemmMaps maps;
    GemmArgs args;
    dim3 grid;
    int smem;
};

// Build the launch plan for sum_{s<n_seg} A_s . B_s with shape M x N x K.
template <int KIND, int BN, bool A_MN, bool B_MN>
GemmPlan plan_gemm(const Operand *A, const Operand *B, int n_seg, int M, int N, int K, int splits, float *ws,
                   int *counters) {
    using C = GemmCfg<KIND, BN, A_MN, B_MN>;
    GemmPlan p{};
    std::memset(&p.maps, 0, sizeof(p.maps));
    for (int s = 0; s < n_seg; ++s) {
        CDP_REQUIRE(A[s].mn_major == A_MN && B[s].mn_major == B_MN, "operand majorness mismatch");
        p.maps.a[s] = operand_map<KIND>(A[s], 128);
        p.maps.b[s] = operand_map<KIND>(B[s], BN);
    }
    const int kb = (K + C::BK - 1) / C::BK;
    const int total = kb * n_seg;
    splits = std::max(1, std::min(splits, total));
    const int per = (total + splits - 1) / splits;
    splits = (total + per - 1) / per;
    p.args = GemmArgs{M, N, kb, n_seg, per, ws, counters, ConvGeom{}};
    p.grid = dim3((M + 127) / 128, (N + BN - 1) / BN, splits);
    p.smem = C::SMEM;
    CDP_REQUIRE(splits == 1 || (ws && counters), "split-K needs a workspace");
    return p;
}

template <int KIND, int BN, bool A_MN, bool B_MN, class Epi, int MODE = GM_PLAIN>
void launch_gemm(const GemmPlan &p, const typename Epi::Params &ep, cudaStream_t st) {
    using C = GemmCfg<KIND, BN, A_MN, B_MN, Epi::kStages, Epi::template pf_bytes<BN>()>;
    static_assert(!Epi::kTile || 128 * (BN + 4) * 4 <= C::STAGES * C::STAGE_BYTES, "tile epilogue staging too big");
    static_assert(C::SMEM <= 227 * 1024, "shared memory budget exceeded");
    auto kern = gemm_tc_kernel<KIND, BN, A_MN, B_MN, Epi, MODE>;
    static bool attr_set = false;
    if (!attr_set) {
        CDP_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, C::SMEM));
        attr_set = true;
    }
    launch_pdl(kern, p.grid, dim3(256), C::SMEM, st, p.maps, p.args, ep);
}

// ---------------------------------------------------------------------------
// Implicit-GEMM convolution plans (gemm_tc_kernel MODE 1-3).

// An NHWC tensor in compute format: element (n, h, w, c) at hi[((n*H + h)*W + w)*ld + c].
struct Nhwc {
    const void *hi = nullptr, *lo = nullptr;
    int ld = 0, C = 0, W = 0, H = 0, N = 0;
};

inline int pow2_ceil(int x) {
    int p = 1;
    while (p < x) p <<= 1;
    return p;
}

// Pixel boxes of `box_pixels` over a [Bn][Ho][Wo] grid (W fastest).
inline ConvGeom conv_geom(int C, int R, int S, int stride, int pad, int Wo, int Ho, int Bn, int box_pixels, int CH) {
    ConvGeom g{};
    g.C = C;
    g.R = R;
    g.S = S;
    g.stride = stride;
    g.pad = pad;
    g.cpt = C / CH;
    g.bw = std::min(box_pixels, pow2_ceil(Wo));
    g.bh = std::min(box_pixels / g.bw, pow2_ceil(Ho));
    g.bn = box_pixels / (g.bw * g.bh);
    g.nbw = (Wo + g.bw - 1) / g.bw;
    g.nbh = (Ho + g.bh - 1) / g.bh;
    g.Wo = Wo;
    g.Ho = Ho;
    g.Bn = Bn;
    g.omul = 1;
    g.oph = g.opw = 0;
    g.oH = Ho;
    g.oW = Wo;
    return g;
}

// Data-gradient taps.  phase < 0: a stride-1 conv, all R*S taps, dx(h, w) <- dy(h + pad - r, w + pad - s).
// phase = ph*2 + pw (stride 2): output pixels (2i + ph, 2j + pw) <- dy(i + (ph + pad - r)/2, ...) over the
// taps with (ph + pad - r) and (pw + pad - s) even.
inline void dgrad_taps(ConvGeom &g, int R, int S, int pad, int phase) {
    g.ntap = 0;
    for (int r = 0; r < R; ++r)
        for (int s = 0; s < S; ++s) {
            int oh, ow;
            if (phase < 0) {
                oh = pad - r;
                ow = pad - s;
            } else {
                const int ph = phase >> 1, pw = phase & 1;
                if (((ph + pad - r) & 1) || ((pw + pad - s) & 1)) continue;
                oh = (ph + pad - r) / 2;
                ow = (pw + pad - s) / 2;
            }
            g.toh[g.ntap] = (signed char)oh;
            g.tow[g.ntap] = (signed char)ow;
            g.twt[g.ntap] = (signed char)(r * S + s);
            ++g.ntap;
        }
}
inline int conv_boxes(const ConvGeom &g) { return g.nbw * g.nbh * ((g.Bn + g.bn - 1) / g.bn); }

// 4-D map over an NHWC tensor; box = CH channels x (bw, bh, bn) pixels at element stride es.
template <int KIND>
CUtensorMap nhwc_map(const void *ptr, const Nhwc &t, int bw, int bh, int bn, int es, bool mn_major) {
    constexpr int ELEM = KIND == 0 ? 2 : 4;
    constexpr uint32_t CH = 128 / ELEM;
    const uint64_t dims[4] = {uint64_t(t.C), uint64_t(t.W), uint64_t(t.H), uint64_t(t.N)};
    const uint64_t rs = uint64_t(t.ld) * ELEM;
    const uint64_t strides[3] = {rs, rs * t.W, rs * t.W * t.H};
    const uint32_t box[4] = {CH, uint32_t(bw * es), uint32_t(bh * es), uint32_t(bn)};
    const uint32_t estr[4] = {1, uint32_t(es), uint32_t(es), 1};
    const CUtensorMapSwizzle swz =
        (mn_major && KIND == 1) ? CU_TENSOR_MAP_SWIZZLE_128B_ATOM_32B : CU_TENSOR_MAP_SWIZZLE_128B;
    return make_tmap_4d(ptr, KIND == 0 ? ElemType::BF16 : ElemType::F32, dims, strides, box, estr, swz);
}

// Segments of the 3xTF32 product (hi.hi + hi.lo + lo.hi); bf16: one segment.
template <int KIND>
inline int seg_pick(int s, bool a) {
    // s: 0 -> (hi, hi), 1 -> (hi, lo), 2 -> (lo, hi); returns 1 for "lo"
    return a ? (s == 2) : (s == 1);
}

// FPROP: out[P_out][Cout] = conv(x, W);  x NHWC (C % CH == 0), W compute copy [R*S*C][Cout].
// DGRAD: dx[P_in][Cin] = conv^T(dy, W) for stride 1;  dy NHWC [.][Cout], W as above.
// WGRAD: dW[R*S*C][Cout] = sum_pixels x_tap^T dy;  x NHWC, dy NHWC.
template <int KIND, int BN, int MODE>
GemmPlan plan_conv(const Nhwc &a, const void *b_hi, const void *b_lo, int b_ld, const Nhwc &dy, int R, int S,
                   int stride, int pad, int Cin, int Cout, int splits, float *ws, int *counters, int phase = -1) {
    constexpr int ELEM = KIND == 0 ? 2 : 4;
    constexpr int CH = 128 / ELEM;
    constexpr bool A_MN = MODE == GM_WGRAD;
    constexpr bool B_MN = MODE != GM_DGRAD;
    using Cfg = GemmCfg<KIND, BN, A_MN, B_MN>;
    const int n_seg = KIND == 0 ? 1 : 3;
    GemmPlan p{};
    std::memset(&p.maps, 0, sizeof(p.maps));
    ConvGeom g{};
    int M = 0, N = 0, kb = 0, tiles_m = 0;
    if (MODE == GM_FPROP) {
        CDP_REQUIRE(a.C % CH == 0 && a.C == Cin, "implicit conv: input channels must be a multiple of the chunk");
        const int Ho = (a.H + 2 * pad - R) / stride + 1, Wo = (a.W + 2 * pad - S) / stride + 1;
        g = conv_geom(Cin, R, S, stride, pad, Wo, Ho, a.N, 128, CH);
        M = a.N * Ho * Wo;
        N = Cout;
        kb = R * S * g.cpt;
        tiles_m = conv_boxes(g);
        for (int s = 0; s < n_seg; ++s) {
            p.maps.a[s] = nhwc_map<KIND>(seg_pick<KIND>(s, true) ? a.lo : a.hi, a, g.bw, g.bh, g.bn, stride, false);
            Operand bo{seg_pick<KIND>(s, false) ? b_lo : b_hi, true, uint64_t(Cout), uint64_t(R * S * Cin),
                       uint64_t(b_ld)};
            p.maps.b[s] = operand_map<KIND>(bo, BN);
        }
    } else if (MODE == GM_DGRAD) {
        CDP_REQUIRE(dy.C % CH == 0 && dy.C == Cout, "implicit dgrad: output channels must be a multiple of the chunk");
        if (stride == 1) {
            CDP_REQUIRE(phase < 0, "stride-1 dgrad has no phases");
            const int H = dy.H + R - 1 - 2 * pad, W = dy.W + S - 1 - 2 * pad;  // forward input extents
            g = conv_geom(Cout, R, S, 1, pad, W, H, dy.N, 128, CH);
            M = dy.N * H * W;
        } else {
            CDP_REQUIRE(stride == 2 && phase >= 0 && phase < 4, "stride-2 dgrad runs as 4 sub-pixel phases");
            CDP_REQUIRE(a.H >= 2 * dy.H - 1 && a.H <= 2 * dy.H && a.W >= 2 * dy.W - 1 && a.W <= 2 * dy.W,
                        "stride-2 dgrad: input extents must be 2*Ho or 2*Ho - 1");
            // phase grid = the dy grid; output pixel (2i + ph, 2j + pw) of the (a.H x a.W) input
            g = conv_geom(Cout, R, S, 2, pad, dy.W, dy.H, dy.N, 128, CH);
            g.omul = 2;
            g.oph = phase >> 1;
            g.opw = phase & 1;
            g.oH = a.H;
            g.oW = a.W;
            M = dy.N * a.H * a.W;
        }
        dgrad_taps(g, R, S, pad, phase);
        CDP_REQUIRE(g.ntap > 0, "empty dgrad phase");
        g.Cw = Cin;
        N = Cin;
        kb = g.ntap * g.cpt;
        tiles_m = conv_boxes(g);
        for (int s = 0; s < n_seg; ++s) {
            p.maps.a[s] = nhwc_map<KIND>(seg_pick<KIND>(s, true) ? dy.lo : dy.hi, dy, g.bw, g.bh, g.bn, 1, false);
            Operand bo{seg_pick<KIND>(s, false) ? b_lo : b_hi, false, uint64_t(R * S * Cin), uint64_t(Cout),
                       uint64_t(b_ld)};
            p.maps.b[s] = operand_map<KIND>(bo, BN);
        }
    } else {
        CDP_REQUIRE(a.C % CH == 0 && a.C == Cin && dy.C == Cout, "implicit wgrad: channel mismatch");
        g = conv_geom(Cin, R, S, stride, pad, dy.W, dy.H, dy.N, Cfg::BK, CH);
        M = R * S * Cin;
        N = Cout;
        kb = conv_boxes(g);
        tiles_m = (M + 127) / 128;
        for (int s = 0; s < n_seg; ++s) {
            p.maps.a[s] = nhwc_map<KIND>(seg_pick<KIND>(s, true) ? a.lo : a.hi, a, g.bw, g.bh, g.bn, stride, true);
            p.maps.b[s] = nhwc_map<KIND>(seg_pick<KIND>(s, false) ? dy.lo : dy.hi, dy, g.bw, g.bh, g.bn, 1, true);
        }
    }
    const int total = kb * n_seg;
    splits = std::max(1, std::min(splits, total));
    const int per = (total + splits - 1) / splits;
    splits = (total + per - 1) / per;
    p.args = GemmArgs{M, N, kb, n_seg, per, ws, counters, g};
    p.grid = dim3(tiles_m, (N + BN - 1) / BN, splits);
    p.smem = Cfg::SMEM;
    CDP_REQUIRE(splits == 1 || (ws && counters), "split-K needs a workspace");
    return p;
}

// Workspace bytes needed by a split-K plan.
inline size_t gemm_ws_floats(const GemmPlan &p, int BN) {
    return p.grid.z > 1 ? size_t(p.grid.x) * p.grid.y * p.grid.z * 128 * BN : 0;
}

}  // namespace cdp
