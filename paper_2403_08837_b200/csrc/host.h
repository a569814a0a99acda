// Host-side helpers shared by the C-ABI translation units: error state,
// CUDA checks, TMA tensor-map encoding through the driver entry point.
#pragma once
#include <cuda.h>
#include <cuda_runtime.h>
#include <stdint.h>

#include <cstdio>
#include <cstdlib>
#include <utility>
#include <stdexcept>
#include <string>

namespace cdp {

void set_error(const std::string &msg);
const char *get_error();

struct CdpError : std::runtime_error {
    explicit CdpError(const std::string &m) : std::runtime_error(m) {}
};

#define CDP_CUDA(expr)                                                                                          \
    do {                                                                                                        \
        cudaError_t e__ = (expr);                                                                               \
        if (e__ != cudaSuccess)                                                                                 \
            throw ::cdp::CdpError(std::string(#expr) + ": " + cudaGetErrorString(e__) + " @" + __FILE__ + ":" + \
                                  std::to_string(__LINE__));                                                    \
    } while (0)

#define CDP_REQUIRE(cond, msg)                               \
    do {                                                     \
        if (!(cond)) throw ::cdp::CdpError(std::string(msg)); \
    } while (0)

// C-ABI guard: run body, convert exceptions to an error code + last-error string.
template <class F>
int guarded(F &&f) {
    try {
        f();
        return 0;
    } catch (const std::exception &e) {
        set_error(e.what());
        return 1;
    } catch (...) {
        set_error("unknown error");
        return 1;
    }
}

enum class ElemType { BF16 = 0, F32 = 1 };

// 2-D tiled tensor map, 128-byte swizzle.  inner/outer extents in elements,
// row stride in bytes (multiple of 16), box {box_inner, box_outer}.
CUtensorMap make_tmap_2d(const void *base, ElemType t, uint64_t inner, uint64_t outer, uint64_t row_stride_bytes,
                         uint32_t box_inner, uint32_t box_outer,
                         CUtensorMapSwizzle swz = CU_TENSOR_MAP_SWIZZLE_128B);

// 4-D tiled tensor map (NHWC activations: dims {C, W, H, N} innermost first),
// strides in bytes for dims 1..3, element strides for dims 1..3 (dim 0 must be 1).
CUtensorMap make_tmap_4d(const void *base, ElemType t, const uint64_t dims[4], const uint64_t strides_bytes[3],
                         const uint32_t box[4], const uint32_t estr[4], CUtensorMapSwizzle swz);

int num_sms();

// Programmatic dependent launch (PDL) toggle: CDP_PDL=0 disables it.
bool pdl_enabled();

// Launch `kern` with the programmatic-stream-serialization attribute so its
// prologue overlaps the tail of the previous kernel on the stream (the kernel
// must call griddepcontrol.wait before touching dependent global memory).
template <class... KArgs, class... Args>
void launch_pdl(void (*kern)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t st, Args &&...args) {
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = grid;
    cfg.blockDim = block;
    cfg.dynamicSmemBytes = smem;
    cfg.stream = st;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = attr;
    cfg.numAttrs = pdl_enabled() ? 1 : 0;
    CDP_CUDA(cudaLaunchKernelEx(&cfg, kern, std::forward<Args>(args)...));
}

// Same, launched as clusters of `cx` CTAs along x.
template <typename... KArgs, typename... Args>
void launch_pdl_cluster(void (*kern)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t st, int cx,
                        Args &&...args) {
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = grid;
    cfg.blockDim = block;
    cfg.dynamicSmemBytes = smem;
    cfg.stream = st;
    cudaLaunchAttribute attr[2];
    attr[0].id = cudaLaunchAttributeClusterDimension;
    attr[0].val.clusterDim.x = unsigned(cx);
    attr[0].val.clusterDim.y = 1;
    attr[0].val.clusterDim.z = 1;
    attr[1].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[1].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = attr;
    cfg.numAttrs = pdl_enabled() ? 2 : 1;
    CDP_CUDA(cudaLaunchKernelEx(&cfg, kern, std::forward<Args>(args)...));
}

// Clusters of `cx` CTAs (block threads, smem bytes) that fit on the GPU at once.
template <typename... KArgs>
int max_active_clusters(void (*kern)(KArgs...), int block, size_t smem, int cx) {
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = dim3(unsigned(cx) * 64);
    cfg.blockDim = dim3(unsigned(block));
    cfg.dynamicSmemBytes = smem;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeClusterDimension;
    attr[0].val.clusterDim.x = unsigned(cx);
    attr[0].val.clusterDim.y = 1;
    attr[0].val.clusterDim.z = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    int n = 0;
    CDP_CUDA(cudaOccupancyMaxActiveClusters(&n, kern, &cfg));
    return n;
}

}  // namespace cdp
