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
    p.args = GemmArgs{M, N, kb, n_seg, per, ws, counters};
    p.grid = dim3((M + 127) / 128, (N + BN - 1) / BN, splits);
    p.smem = C::SMEM;
    CDP_REQUIRE(splits == 1 || (ws && counters), "split-K needs a workspace");
    return p;
}

template <int KIND, int BN, bool A_MN, bool B_MN, class Epi>
void launch_gemm(const GemmPlan &p, const typename Epi::Params &ep, cudaStream_t st) {
    using C = GemmCfg<KIND, BN, A_MN, B_MN, Epi::kStages, Epi::template pf_bytes<BN>()>;
    static_assert(!Epi::kTile || 128 * (BN + 4) * 4 <= C::STAGES * C::STAGE_BYTES, "tile epilogue staging too big");
    static_assert(C::SMEM <= 227 * 1024, "shared memory budget exceeded");
    auto kern = gemm_tc_kernel<KIND, BN, A_MN, B_MN, Epi>;
    static bool attr_set = false;
    if (!attr_set) {
        CDP_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, C::SMEM));
        attr_set = true;
    }
    launch_pdl(kern, p.grid, dim3(256), C::SMEM, st, p.maps, p.args, ep);
}

// Workspace bytes needed by a split-K plan.
inline size_t gemm_ws_floats(const GemmPlan &p, int BN) {
    return p.grid.z > 1 ? size_t(p.grid.x) * p.grid.y * p.grid.z * 128 * BN : 0;
}

}  // namespace cdp
