#include <mutex>

#include "host.h"

namespace cdp {

static thread_local std::string g_err;

void set_error(const std::string &msg) { g_err = msg; }
const char *get_error() { return g_err.c_str(); }

typedef CUresult (*PFN_encodeTiled_t)(CUtensorMap *, CUtensorMapDataType, cuuint32_t, void *, const cuuint64_t *,
                                      const cuuint64_t *, const cuuint32_t *, const cuuint32_t *,
                                      CUtensorMapInterleave, CUtensorMapSwizzle, CUtensorMapL2promotion,
                                      CUtensorMapFloatOOBfill);

static PFN_encodeTiled_t encode_fn() {
    static PFN_encodeTiled_t fn = nullptr;
    static std::once_flag once;
    std::call_once(once, [] {
        void *p = nullptr;
        cudaDriverEntryPointQueryResult q;
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
            q == cudaDriverEntryPointSuccess)
            fn = reinterpret_cast<PFN_encodeTiled_t>(p);
    });
    CDP_REQUIRE(fn != nullptr, "cuTensorMapEncodeTiled entry point unavailable");
    return fn;
}

CUtensorMap make_tmap_2d(const void *base, ElemType t, uint64_t inner, uint64_t outer, uint64_t row_stride_bytes,
                         uint32_t box_inner, uint32_t box_outer, CUtensorMapSwizzle swz) {
    CUtensorMap m;
    cuuint64_t dims[2] = {inner, outer};
    cuuint64_t strides[1] = {row_stride_bytes};
    cuuint32_t box[2] = {box_inner, box_outer};
    cuuint32_t estr[2] = {1, 1};
    CDP_REQUIRE(row_stride_bytes % 16 == 0, "TMA row stride must be a multiple of 16 bytes");
    CDP_REQUIRE((reinterpret_cast<uintptr_t>(base) & 15) == 0, "TMA base must be 16-byte aligned");
    CUresult r = encode_fn()(&m, t == ElemType::BF16 ? CU_TENSOR_MAP_DATA_TYPE_BFLOAT16 : CU_TENSOR_MAP_DATA_TYPE_FLOAT32,
                             2, const_cast<void *>(base), dims, strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
                             swz, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                             CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    CDP_REQUIRE(r == CUDA_SUCCESS, "cuTensorMapEncodeTiled failed (code " + std::to_string(int(r)) + ")");
    return m;
}

CUtensorMap make_tmap_4d(const void *base, ElemType t, const uint64_t dims_in[4], const uint64_t strides_bytes[3],
                         const uint32_t box_in[4], const uint32_t estr_in[4], CUtensorMapSwizzle swz) {
    CUtensorMap m;
    cuuint64_t dims[4], strides[3];
    cuuint32_t box[4], estr[4];
    for (int i = 0; i < 4; ++i) {
        dims[i] = dims_in[i];
        box[i] = box_in[i];
        estr[i] = estr_in[i];
        CDP_REQUIRE(box[i] >= 1 && box[i] <= 256, "TMA box dimension out of range");
        CDP_REQUIRE(estr[i] >= 1 && estr[i] <= 8, "TMA element stride out of range");
    }
    for (int i = 0; i < 3; ++i) {
        strides[i] = strides_bytes[i];
        CDP_REQUIRE(strides[i] % 16 == 0, "TMA strides must be multiples of 16 bytes");
    }
    CDP_REQUIRE((reinterpret_cast<uintptr_t>(base) & 15) == 0, "TMA base must be 16-byte aligned");
    CUresult r = encode_fn()(&m, t == ElemType::BF16 ? CU_TENSOR_MAP_DATA_TYPE_BFLOAT16 : CU_TENSOR_MAP_DATA_TYPE_FLOAT32,
                             4, const_cast<void *>(base), dims, strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE, swz,
                             CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    CDP_REQUIRE(r == CUDA_SUCCESS, "cuTensorMapEncodeTiled (4-D) failed (code " + std::to_string(int(r)) + ")");
    return m;
}

bool pdl_enabled() {
    static const bool on = [] {
        const char *e = std::getenv("CDP_PDL");
        return !(e && e[0] == '0');
    }();
    return on;
}

int num_sms() {
    int dev = 0, n = 0;
    CDP_CUDA(cudaGetDevice(&dev));
    CDP_CUDA(cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev));
    return n;
}

}  // namespace cdp
