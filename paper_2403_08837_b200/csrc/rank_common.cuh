// Kernels and helpers shared by the one-worker-per-process trainers (ResNet, ViT):
// parameter pulls from the updater (the theta delivery of SURVEY §5), the step
// bookkeeping kernel, compute-copy packing, and the GEMM tile-width dispatch.
#pragma once
#include <string>
#include <type_traits>

#include "conv_kernels.cuh"
#include "trainer_common.cuh"

namespace cdp {
namespace {

// Wait (one thread) until the updater holds the version this rank reads of `unit`.
__global__ void pull_wait_kernel(RingFlags *updater, RingFlags *own, int unit, int fresh, const int *step) {
    const int t = *step;
    const uint32_t v = uint32_t(fresh ? t : t - 1);
    if (v > 1 && threadIdx.x == 0) spin_ge(&updater->updated[unit - 1], v, &own->err);
}

// ---------------------------------------------------------------- trace mode (tests)
// Every theta slot carries a version tag (RingFlags::vtag) written by whoever writes the slot's
// data: set_params (host), the update (vtag_update_kernel after the update kernel on the same
// stream), a pull (copies the updater's tag while the updater is still held off by `pulled`), a
// ZeRO-CDP state copy (copies the predecessor's tags).  Around every read of a unit's parameters an
// access record (step, rank, unit, kind, phase, slot, tag) is appended: the executed-version trace
// of ref engine.py:92-94, made from the data actually present in the slot the kernel reads.
enum AccessKind { A_FWD = 0, A_BWD = 1, A_UPD = 2, A_NEW = 3 };
constexpr int kTraceWords = 8;

struct TraceLog {
    uint32_t *rec;
    uint32_t *cursor;
    uint32_t cap;
};

__global__ void access_record_kernel(TraceLog lg, const RingFlags *own, int rank, int unit, int kind, int phase,
                                     int slot, const int *step) {
    const uint32_t i = atomicAdd(lg.cursor, 1u);
    if (i >= lg.cap) return;
    uint32_t *r = lg.rec + size_t(i) * kTraceWords;
    r[0] = uint32_t(*step);
    r[1] = uint32_t(rank);
    r[2] = uint32_t(unit);
    r[3] = uint32_t(kind);
    r[4] = uint32_t(phase);
    r[5] = uint32_t(slot);
    r[6] = ptx::ld_acquire_sys(&own->vtag[slot][unit - 1]);
    r[7] = 0;
}

// After the update of `unit` at step t (same stream): its new slot holds version t + 1.
__global__ void vtag_update_kernel(RingFlags *own, int unit, const int *step) {
    const uint32_t t = uint32_t(*step);
    __threadfence_system();
    ptx::st_release_sys(&own->vtag[(t + 1) & 1][unit - 1], t + 1);
}

// ---------------------------------------------------------------- peer state copies
// Copy of one parameter tensor's state from peer HBM (NVLink when the ranks are GPUs): up to
// three fp32 arrays (theta slots, momentum) of the tensor's [rows][cols] flat layout, and the
// compute-format packing of the first two into their GEMM copies (bf16 / fp32 hi+lo rows of
// pitch wc.ld).  16-byte volatile loads (the peer rewrites the slot between steps), every load
// of an element group issued before its stores, and no per-element index arithmetic beyond an
// add: a thread's (row offset, column quad) is fixed for the whole loop (one division per thread
// at entry).  Rows of <= 4 * blockDim columns are packed several per block pass; wider rows loop
// over their columns; tensors whose rows are not float4-aligned (the 10-class classifier) or
// flat vectors without a packed copy fall back to the scalar / flat paths.
struct StateCopy {
    const float *src[3];
    float *dst[3];
    int narr;
    CTensor wc[2];  // wc[k].hi: pack array k into it
    int64_t n;
    int cols;
};

template <int KIND>
__device__ __forceinline__ void state_copy_quad(const StateCopy &c, size_t o, size_t ow) {
    float4 x[3];
#pragma unroll
    for (int k = 0; k < 3; ++k)
        if (k < c.narr) x[k] = __ldcv(reinterpret_cast<const float4 *>(c.src[k] + o));
#pragma unroll
    for (int k = 0; k < 3; ++k)
        if (k < c.narr) {
            *reinterpret_cast<float4 *>(c.dst[k] + o) = x[k];
            if (k < 2 && c.wc[k].hi) store_wc4<KIND>(c.wc[k], ow, x[k]);
        }
}

template <int KIND>
__device__ void state_copy(const StateCopy &c) {
    bool aligned = (c.n & 3) == 0;
#pragma unroll
    for (int k = 0; k < 3; ++k)
        if (k < c.narr)
            aligned = aligned && ((reinterpret_cast<uintptr_t>(c.src[k]) | reinterpret_cast<uintptr_t>(c.dst[k])) & 15) == 0;
    const bool packed = c.wc[0].hi || c.wc[1].hi;
    if (aligned && !packed) {  // flat vector (batch-norm gamma | beta): float4 over the flat range
        const int64_t n4 = c.n / 4;
        for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < n4; i += int64_t(gridDim.x) * blockDim.x)
            state_copy_quad<KIND>(c, size_t(i) * 4, 0);
        return;
    }
    if (aligned && (c.cols & 3) == 0 && (c.wc[0].ld & 3) == 0 && (c.wc[1].ld & 3) == 0) {
        const int q = c.cols / 4;
        const int64_t rows = c.n / c.cols;
        if (q <= int(blockDim.x)) {
            const int rpb = blockDim.x / q;
            const int r0 = threadIdx.x / q, c4 = (threadIdx.x - r0 * q) * 4;
            if (r0 >= rpb) return;
            for (int64_t r = blockIdx.x * int64_t(rpb) + r0; r < rows; r += int64_t(gridDim.x) * rpb)
                state_copy_quad<KIND>(c, size_t(r) * c.cols + c4, size_t(r) * c.wc[0].ld + c4);
        } else {
            for (int64_t r = blockIdx.x; r < rows; r += gridDim.x)
                for (int c4 = threadIdx.x * 4; c4 < c.cols; c4 += blockDim.x * 4)
                    state_copy_quad<KIND>(c, size_t(r) * c.cols + c4, size_t(r) * c.wc[0].ld + c4);
        }
        return;
    }
    for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < c.n; i += int64_t(gridDim.x) * blockDim.x) {
        const size_t w = size_t(i / c.cols) * c.wc[0].ld + i % c.cols;
#pragma unroll
        for (int k = 0; k < 3; ++k)
            if (k < c.narr) {
                const float x = __ldcv(c.src[k] + i);
                c.dst[k][i] = x;
                if (k < 2 && c.wc[k].hi) Fmt<KIND>::store(c.wc[k].hi, c.wc[k].lo, w, x);
            }
    }
}

template <int KIND>
__global__ void pull_tensor_kernel(const float *__restrict__ src, float *dst, int64_t n, int cols, CTensor wc,
                                   RingFlags *updater, RingFlags *own, int unit, int fresh, const int *step,
                                   unsigned *cta_counter, int trace) {
    ptx::griddep_wait();
    ptx::griddep_launch();
    const int t = *step;
    const uint32_t v = uint32_t(fresh ? t : t - 1);
    if (v <= 1) return;
    StateCopy c{};
    c.src[0] = src;
    c.dst[0] = dst;
    c.narr = 1;
    c.wc[0] = wc;
    c.n = n;
    c.cols = cols;
    state_copy<KIND>(c);
    __syncthreads();
    if (threadIdx.x == 0) {
        __threadfence_system();
        if (atomicAdd(&cta_counter[unit - 1], 1u) == gridDim.x - 1) {
            cta_counter[unit - 1] = 0;
            // the updater cannot overwrite slot v & 1 before this arrival: its tag is the copied version
            if (trace) own->vtag[v & 1][unit - 1] = ptx::ld_acquire_sys(&updater->vtag[v & 1][unit - 1]);
            atomicAdd_system(&updater->pulled[unit - 1][v & 1], 1u);
        }
    }
}

// ---------------------------------------------------------------- theta forwarding along the readers
// The readers of version v of a unit pull it in the order they read it (the reader order of the rule:
// fresh readers in worker order at step v, then stale readers at step v + 1); the first takes it from
// the updater, each later one from the reader before it, so every rank serves one copy per version
// instead of the updater serving all N - 1 (the egress hot spot of the N - 1 pulls from rank N - 1).
// A reader overwrites its slot v & 1 with v + 2 only after its successor took v from it.
__global__ void chain_wait_kernel(const RingFlags *pred, int pred_is_updater, RingFlags *own, int unit, int fresh,
                                  int has_succ, const int *step) {
    const int t = *step;
    const uint32_t v = uint32_t(fresh ? t : t - 1);
    if (v <= 1 || threadIdx.x != 0) return;
    if (pred_is_updater)
        spin_ge(&pred->updated[unit - 1], v, &own->err);
    else
        spin_ge(&pred->fwd_have[unit - 1], v, &own->err);
    if (has_succ && v > 3) spin_ge(&own->fwd_pulled[unit - 1][v & 1], v - 2, &own->err);
}

template <int KIND>
__global__ void chain_pull_kernel(const float *__restrict__ src, float *dst, int64_t n, int cols, CTensor wc,
                                  RingFlags *pred, int pred_is_updater, RingFlags *own, int unit, int fresh,
                                  const int *step, unsigned *cta_counter, int trace) {
    ptx::griddep_wait();
    ptx::griddep_launch();
    const int t = *step;
    const uint32_t v = uint32_t(fresh ? t : t - 1);
    if (v <= 1) return;
    StateCopy c{};
    c.src[0] = src;
    c.dst[0] = dst;
    c.narr = 1;
    c.wc[0] = wc;
    c.n = n;
    c.cols = cols;
    state_copy<KIND>(c);
    __syncthreads();
    if (threadIdx.x == 0) {
        __threadfence_system();
        if (atomicAdd(&cta_counter[unit - 1], 1u) == gridDim.x - 1) {
            cta_counter[unit - 1] = 0;
            // the source cannot overwrite slot v & 1 before this arrival: its tag is the copied version
            if (trace) own->vtag[v & 1][unit - 1] = ptx::ld_acquire_sys(&pred->vtag[v & 1][unit - 1]);
            __threadfence_system();
            ptx::st_release_sys(&own->fwd_have[unit - 1], v);
            if (pred_is_updater)
                atomicAdd_system(&pred->pulled[unit - 1][v & 1], 1u);
            else
                ptx::st_release_sys(&pred->fwd_pulled[unit - 1][v & 1], v);
        }
    }
}

__global__ void finish_step_kernel_rn(const double *loss, Flags *flags, double *hist_loss, Flags *hist_flags, int cap,
                                      const int *step) {
    const int c = *step - 1;
    hist_loss[c % cap] = *loss;
    hist_flags[c % cap] = *flags;
    *flags = Flags{0, 0, 0, 0};
}

template <int KIND>
__global__ void pack_tensor_kernel(const float *__restrict__ w, int64_t n, int cols, CTensor out) {
    for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < n; i += int64_t(gridDim.x) * blockDim.x)
        Fmt<KIND>::store(out.hi, out.lo, size_t(i / cols) * out.ld + i % cols, w[i]);
}

template <int V>
using IC = std::integral_constant<int, V>;

template <class F>
void bn_switch(int BN, F &&f) {
    switch (BN) {
        case 32: f(IC<32>{}); return;
        case 64: f(IC<64>{}); return;
        case 128: f(IC<128>{}); return;
        case 256: f(IC<256>{}); return;
        default: throw CdpError("unsupported GEMM tile width " + std::to_string(BN));
    }
}

}  // namespace
}  // namespace cdp
