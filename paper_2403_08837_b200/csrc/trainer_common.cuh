// Infrastructure shared by the device trainers: owning device buffers,
// compute-format tensors, the per-step control block and flag words.
#pragma once
#include <algorithm>
#include <utility>

#include "host.h"
#include "mlp_kernels.cuh"

namespace cdp {

inline int round_up(int x, int m) { return (x + m - 1) / m * m; }

struct DevBuf {
    void *p = nullptr;
    size_t bytes = 0;
    DevBuf() = default;
    explicit DevBuf(size_t b) : bytes(b) {
        if (b) {
            CDP_CUDA(cudaMalloc(&p, b));
            CDP_CUDA(cudaMemset(p, 0, b));
        }
    }
    DevBuf(const DevBuf &) = delete;
    DevBuf &operator=(const DevBuf &) = delete;
    DevBuf(DevBuf &&o) noexcept : p(o.p), bytes(o.bytes) { o.p = nullptr; o.bytes = 0; }
    DevBuf &operator=(DevBuf &&o) noexcept {
        std::swap(p, o.p);
        std::swap(bytes, o.bytes);
        return *this;
    }
    ~DevBuf() {
        if (p) cudaFree(p);
    }
    template <class T>
    T *as() const { return static_cast<T *>(p); }
};

// A compute-format tensor [rows][ld] (two arrays for 3xTF32).
struct CBuf {
    DevBuf hi, lo;
    int ld = 0;
    CTensor view() const { return CTensor{hi.p, lo.p, ld}; }
};

inline CBuf make_cbuf(int kind, int rows, int cols) {
    CBuf b;
    const int esz = kind == 0 ? 2 : 4;
    b.ld = round_up(std::max(cols, 1), 16);  // 16-element rows keep TMA strides 16B-aligned
    b.hi = DevBuf(size_t(rows) * b.ld * esz);
    if (kind == 1) b.lo = DevBuf(size_t(rows) * b.ld * esz);
    return b;
}

struct Control {  // device control block, refreshed from pinned host memory every step
    float lr;
    int step;
    int pad[2];
};

struct Flags {
    unsigned grad, loss, upd, pad;
};

static __global__ void stamp_kernel(uint64_t *out) {
    uint64_t t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    *out = t;
}

}  // namespace cdp
