// Device-resident CDP training step for ResNets (BASELINE configs[1..2,4]):
// BasicBlock or Bottleneck residual stages, CIFAR stem (3x3/s1) or ImageNet
// stem (7x7/s2 + 3x3/s2 max pool), one micro-batch per GPU.
//
// Same step semantics as the MLP trainer (ref training/engine.py:66-116 with
// the per-stage version rule, gradient hops w_i -> w_{i+1}, fused update on
// the last worker, parameter pulls) with convolutional layer compute:
//   conv fprop = tcgen05 implicit GEMM: TMA gathers NHWC pixel boxes of the
//                input per filter tap (element strides, OOB zero fill = padding);
//                epilogue writes y and the per-tile BN statistics;
//   BN         = training-mode batch statistics (fp64 fixed-order finalise),
//                affine + residual + ReLU in one vectorised pass;
//   dgrad      = implicit GEMM over dy (stride 1), or four sub-pixel phases of
//                stride-1 implicit GEMMs with the phase's taps (stride 2);
//   wgrad      = implicit GEMM (K = pixel boxes, split-K) whose epilogue is the
//                hop / SGD update of the weight tensor (EpiWgrad);
//   BN gamma|beta hop / update by a vector kernel.
// Hop units are parameter tensors in torchvision order: conv weights
// [R*S*Cin][Cout], BN [gamma(C) | beta(C)], classifier [[W^T]; b] = [C+1][classes].
#include <cuda_bf16.h>

#include <cstdlib>
#include <cstring>
#include <functional>
#include <memory>
#include <string>
#include <type_traits>
#include <vector>

#include "../../include/cdp_b200.h"
#include "conv_kernels.cuh"
#include "gemm_launch.cuh"
#include "trainer_common.cuh"
#include "rank_common.cuh"

namespace cdp {

namespace {

enum TensorKind { T_CONV = 0, T_BN = 1, T_FC = 2 };
enum ConvImpl { CI_IMPLICIT = 0, CI_PLAIN = 1, CI_STEM = 2 };

struct TensorSpec {
    int kind;
    int64_t base, n;
    int rows, cols;  // GEMM view for conv / fc
    int stage;       // 1-based stage (version unit)
    int fresh;       // this worker reads the current version of this tensor's stage
};

struct ConvL {
    int cin, cout, R, S, stride, pad, H, W, Ho, Wo, K;
    int impl;
    int tw, tb;        // tensor indices of the weight and its BN
    int in_act;        // activation index of the input (-1: the stem's im2col record)
    int64_t P, Pin;    // output / input pixels
    int tiles_fwd;     // M tiles of the forward GEMM (rows of the BN statistics)
    DevBuf y, mean, rstd, dbeta, dgamma;
    CBuf dy;           // gradient w.r.t. the conv output (GEMM operand)
};

struct BlockL {
    std::vector<int> convs;  // main path
    std::vector<int> mid;    // activation after convs[i] (i < n-1)
    int ds = -1;             // projection shortcut conv (-1: identity)
    int a_in = 0, a_out = 0;
};

struct OpRec {
    std::string name;
    double flops, bytes;
    cudaEvent_t a, b;
};

// ---------------------------------------------------------------- ZeRO-CDP state passing
// (zero.py: use index u = base + (t-1)*2N + kZeroOff; predecessor on rank `src` in step t + dstep)
constexpr uint32_t kZeroOff = 1024;

struct ZeroUse {
    int base, src, dstep, uses_per_step;
};

__device__ __forceinline__ uint32_t zero_u(const ZeroUse &z, int t) {
    return uint32_t(z.base + (t - 1) * z.uses_per_step) + kZeroOff;
}

// Wait (one thread) until the predecessor's rank finished its use of `unit`.
__global__ void zero_wait_kernel(ZeroUse z, int self, const RingFlags *src_flags, RingFlags *own, int unit,
                                 const int *step, int step_delta, int copy_tags) {
    const int t = *step + step_delta;
    if (threadIdx.x != 0 || z.src == self || t + z.dstep < 1) return;
    const uint32_t pu = zero_u(z, t) - 1;
    spin_ge(&src_flags->zdone[unit - 1], pu, &own->err);
    if (copy_tags) {  // trace mode: the state copy that follows brings the predecessor's versions
        own->vtag[0][unit - 1] = ptx::ld_acquire_sys(&src_flags->vtag[0][unit - 1]);
        own->vtag[1][unit - 1] = ptx::ld_acquire_sys(&src_flags->vtag[1][unit - 1]);
    }
}

// Copy the unit's state (both theta version slots, momentum) from the predecessor's HBM
// (peer memory) and repack the compute copies of both slots.
// ZeRO-CDP frames: a use without predecessor (step 1) loads the initial state from mapped host
// memory (init_t: theta, init_v: zeros) into the frame; with full replicas (init_t null) every rank
// already holds it.
template <int KIND>
__global__ void zero_copy_kernel(ZeroUse z, int self, const float *src_t0, const float *src_t1, const float *src_v,
                                 float *t0, float *t1, float *v, int64_t n, int cols, CTensor wc0, CTensor wc1,
                                 const int *step, const float *init_t, const float *init_v) {
    ptx::griddep_wait();
    ptx::griddep_launch();
    const int t = *step;
    const bool initial = t + z.dstep < 1;
    if (initial ? init_t == nullptr : z.src == self) return;
    StateCopy c{};
    c.src[0] = initial ? init_t : src_t0;
    c.src[1] = initial ? init_t : src_t1;
    c.src[2] = initial ? init_v : src_v;
    c.dst[0] = t0;
    c.dst[1] = t1;
    c.dst[2] = v;
    c.narr = v ? 3 : 2;
    c.wc[0] = wc0;
    c.wc[1] = wc1;
    c.n = n;
    c.cols = cols;
    state_copy<KIND>(c);  // rank_common.cuh: 16-byte peer loads, no per-element division
}

// ZeRO-CDP frames: tell the predecessor its copy of `unit` has been taken (its frame may be reused).
__global__ void zero_copied_kernel(ZeroUse z, int self, RingFlags *src_flags, int unit, const int *step) {
    const int t = *step;
    if (z.src == self || t + z.dstep < 1) return;
    __threadfence_system();
    ptx::st_release_sys(&src_flags->zcopied[unit - 1], zero_u(z, t));
}

// ZeRO-CDP frames: before a window copies a stage into a frame, the stage that used the frame two
// windows earlier (use index base_last of step t + dl) must have been copied out by its successor
// (use index + 1, in step t + dl + delta) — when both uses exist.
struct FrameWait {
    int unit0, unit1;  // units (tensor + 1) of the previous occupant
    int base_last, dl, delta, uses_per_step;
};
__global__ void zero_frame_wait_kernel(FrameWait f, RingFlags *own, const int *step) {
    const int t = *step;
    if (threadIdx.x != 0 || t + f.dl < 1 || t + f.dl + f.delta < 1) return;
    const uint32_t want = uint32_t(f.base_last + (t + f.dl - 1) * f.uses_per_step) + kZeroOff + 1;
    for (int u = f.unit0; u < f.unit1; ++u) spin_ge(&own->zcopied[u - 1], want, &own->err);
}

// Publish the end of this rank's use of `unit` (after all its kernels on the stream).
__global__ void zero_done_kernel(ZeroUse z, RingFlags *own, int unit, const int *step, int step_delta) {
    const int t = *step + step_delta;
    __threadfence_system();
    ptx::st_release_sys(&own->zdone[unit - 1], zero_u(z, t));
}

}  // namespace

struct ResNetTrainer {
    // ---------------------------------------------------------------- config
    int kind = 0, B = 0, Hin = 32, Win = 32, Cin0 = 3, classes = 10, loss_kind = 1;
    int block_kind = 0, stem_kind = 0;
    float momentum = 0.f, wd = 0.f, eps = 1e-5f;
    int rank = 0, world = 1;
    std::vector<TensorSpec> tens;
    std::vector<ConvL> convs;
    std::vector<BlockL> blocks;
    int stem = 0, fc_t = -1, fc_in = 0;
    int stem_act = 0, pool_act = -1;  // ImageNet stem: conv output act, max-pool output act
    int64_t P = 0, Pp = 0;

    // ---------------------------------------------------------------- state
    DevBuf region, cta_counters;
    float *vel = nullptr;  // momentum, inside the shared region (ZeRO-CDP peers copy it)
    float *theta[2] = {nullptr, nullptr};
    float *partial = nullptr;
    RingFlags *ring = nullptr;
    size_t region_off = 0;
    RingFlags *prev_ring = nullptr, *upd_ring = nullptr;
    float *prev_partial = nullptr, *upd_theta[2] = {nullptr, nullptr};
    std::vector<CBuf> wc[2];   // per tensor (empty CBuf for BN); full-replica mode
    std::vector<CTensor> wcv[2];  // per tensor: the GEMM compute copy of theta slot v (a frame view in ZeRO mode)
    // ZeRO-CDP frames: a rank keeps the state (theta slots, momentum, compute copies) of only the stages it
    // is using.  Stage s lives in frame (s - 1) & 1 at stage-relative offsets; a rank's consecutive
    // use windows alternate frames (zero.py), so two frames of the largest stage replace the full replica.
    bool frames = false;
    int64_t framePp[2] = {0, 0}, th_stride = 0;  // floats per frame (largest stage of its parity); per slot
    std::vector<int64_t> foff;                   // per tensor: float offset inside a theta slot
    std::vector<int64_t> stage_lo, stage_hi;     // per stage: parameter range [lo, hi)
    std::vector<int> stage_t0, stage_t1;         // per stage: tensor range
    DevBuf wcpool[2][2];                         // [slot][hi / lo] compute-copy frames
    float *init_host = nullptr;                  // mapped pinned: initial theta | zeros (step-1 state source)
    const float *init_dev = nullptr;             // its device alias
    const int32_t *stage_in = nullptr;           // tensor -> stage, set before build()
    std::vector<int> zwin_done;                  // per (stage, kind): frame wait recorded in this step
    std::vector<int> zdrain;                     // end-of-run drain plan rows (zero.py frame_drain_plan)
    std::vector<int> chain;                      // pull chain per stage: (predecessor rank or -1 = updater,
                                                 // successor rank or -1); empty: every reader pulls from the updater
    bool drained = false;                        // frames: a drained run cannot continue
    std::vector<CBuf> acts;    // activations (compute format)
    std::vector<int> act_C, act_H, act_W;
    std::vector<int64_t> act_P;
    DevBuf gbuf[4];            // fp32 gradients w.r.t. activations (block in / chain / chain / shortcut)
    CBuf cols, pooled, dz;     // stem im2col record, pooled features (+ ones column), dZ
    DevBuf dpooled, z, loss_dev, loss_rows, stats_fwd, bnpart[2], pool_arg;
    int64_t max_act = 0;
    DevBuf ws_c, cnt_c, ws_h, cnt_h;
    size_t ws_c_floats = 0, ws_h_floats = 0;
    DevBuf data_x, data_lab, ctrl_dev, perm_dev, flags_dev, hist_loss, hist_flags;
    int n_samples = 0;
    bool allreduce = false;  // DP all-reduce baseline: gradients only, NCCL sum + apply_update on the host side
    // ZeRO-CDP: per (stage, kind F/B, rank) use table from zero.py; peers' shared regions
    bool zero = false;
    std::vector<int> ztab;  // [stages][2][world][3] = (base, src rank, dstep)
    std::vector<uint8_t *> peers;
    int64_t zero_bytes_per_step = 0;
    static constexpr int RING_N = 16;
    uint8_t *stage_host = nullptr;
    size_t stage_bytes = 0;
    cudaEvent_t stage_ev[RING_N] = {};
    int stage_next = 0;
    int hist_cap = 1 << 14;
    cudaStream_t main = nullptr, cs = nullptr, hs = nullptr, ps = nullptr;  // ps: parameter pulls (run ahead)
    cudaStream_t cps = nullptr;           // pipelined input copies (step_host_batch_async)
    cudaEvent_t in_ev[2] = {}, done_ev[2] = {};
    double *loss_host = nullptr;          // pinned: the losses the pipelined steps read back
    std::vector<cudaEvent_t> events;
    cudaGraphExec_t exec[2] = {nullptr, nullptr};
    int t = 1;
    int kernels_per_step = 0;
    double flops_per_step = 0.0;
    std::vector<cudaEvent_t> marks;
    DevBuf flush_buf;
    bool sizing = false;       // dry run: size the split-K workspaces, launch nothing
    bool instr = false;        // eager instrumented step: events around every launch
    bool trace = false;        // version tags + per-access records (tests; rank_common.cuh)
    DevBuf tlog, tcur;
    static constexpr uint32_t kTraceCap = 1u << 16;
    std::vector<OpRec> oprecs;

    ~ResNetTrainer() {
        for (auto &e : exec)
            if (e) cudaGraphExecDestroy(e);
        for (auto e : events) cudaEventDestroy(e);
        for (auto e : marks) cudaEventDestroy(e);
        clear_oprecs();
        for (auto e : stage_ev)
            if (e) cudaEventDestroy(e);
        if (stage_host) cudaFreeHost(stage_host);
        if (init_host) cudaFreeHost(init_host);
        for (auto e : {in_ev[0], in_ev[1], done_ev[0], done_ev[1]})
            if (e) cudaEventDestroy(e);
        if (loss_host) cudaFreeHost(loss_host);
        for (auto s : {main, cs, hs, ps, cps})
            if (s) cudaStreamDestroy(s);
    }

    void clear_oprecs() {
        for (auto &o : oprecs) {
            cudaEventDestroy(o.a);
            cudaEventDestroy(o.b);
        }
        oprecs.clear();
    }

    // Every launch of the step goes through here: counts kernels / flops and,
    // in an instrumented step, brackets the launch with timing events.
    template <class F>
    void L(const char *name, double flops, double bytes, cudaStream_t s, F &&f) {
        if (sizing) return;
        cudaEvent_t a = nullptr, b = nullptr;
        if (instr) {
            CDP_CUDA(cudaEventCreate(&a));
            CDP_CUDA(cudaEventCreate(&b));
            CDP_CUDA(cudaEventRecord(a, s));
        }
        f();
        ++kernels_per_step;
        flops_per_step += flops;
        if (instr) {
            CDP_CUDA(cudaEventRecord(b, s));
            oprecs.push_back(OpRec{name, flops, bytes, a, b});
        }
    }

    // ---------------------------------------------------------------- model
    int chunk() const { return kind == 0 ? 64 : 32; }

    int add_tensor(int k, int64_t n, int rows, int cols_) {
        int64_t base = tens.empty() ? 0 : tens.back().base + tens.back().n;
        tens.push_back(TensorSpec{k, base, n, rows, cols_, 1, 1});
        return int(tens.size()) - 1;
    }

    int add_act(int H, int W, int C) {
        const int64_t rows = int64_t(B) * H * W;
        acts.push_back(make_cbuf(kind, int(rows), C));
        act_C.push_back(C);
        act_H.push_back(H);
        act_W.push_back(W);
        act_P.push_back(rows);
        max_act = std::max(max_act, rows * C);
        return int(acts.size()) - 1;
    }

    int add_conv(int cin, int cout, int R, int stride, int H, int W, int in_act) {
        ConvL c{};
        c.cin = cin;
        c.cout = cout;
        c.R = c.S = R;
        c.stride = stride;
        c.pad = R / 2;
        c.H = H;
        c.W = W;
        c.Ho = (H + 2 * c.pad - R) / stride + 1;
        c.Wo = (W + 2 * c.pad - R) / stride + 1;
        c.K = R * R * cin;
        c.P = int64_t(B) * c.Ho * c.Wo;
        c.Pin = int64_t(B) * H * W;
        c.in_act = in_act;
        c.impl = in_act < 0 ? CI_STEM : (R == 1 && stride == 1) ? CI_PLAIN : CI_IMPLICIT;
        if (c.impl == CI_IMPLICIT) CDP_REQUIRE(cin % chunk() == 0, "conv input channels must fill a TMA chunk");
        c.tw = add_tensor(T_CONV, int64_t(c.K) * cout, c.K, cout);
        c.tb = add_tensor(T_BN, 2 * int64_t(cout), 0, 0);
        if (c.impl == CI_IMPLICIT) {
            const ConvGeom g = conv_geom(cin, R, R, stride, c.pad, c.Wo, c.Ho, B, 128, chunk());
            c.tiles_fwd = conv_boxes(g);
        } else {
            c.tiles_fwd = int((c.P + 127) / 128);
        }
        convs.push_back(std::move(c));
        return int(convs.size()) - 1;
    }

    // Parameter-state layout: full replica (foff = base) or ZeRO-CDP frames (stage-relative offsets).
    void layout_state() {
        foff.resize(tens.size());
        th_stride = Pp;
        for (size_t i = 0; i < tens.size(); ++i) foff[i] = tens[i].base;
        if (!frames) return;
        const int ns = world;
        stage_lo.assign(ns, INT64_MAX);
        stage_hi.assign(ns, 0);
        stage_t0.assign(ns, INT32_MAX);
        stage_t1.assign(ns, 0);
        for (size_t i = 0; i < tens.size(); ++i) {
            const int s = tens[i].stage - 1;
            CDP_REQUIRE(s >= 0 && s < ns, "ZeRO-CDP frames: tensor stage out of range");
            stage_lo[s] = std::min(stage_lo[s], tens[i].base);
            stage_hi[s] = std::max(stage_hi[s], tens[i].base + tens[i].n);
            stage_t0[s] = std::min(stage_t0[s], int(i));
            stage_t1[s] = std::max(stage_t1[s], int(i) + 1);
        }
        framePp[0] = framePp[1] = 0;
        for (int s = 0; s < ns; ++s) {
            CDP_REQUIRE(stage_t1[s] > stage_t0[s], "ZeRO-CDP frames: a stage without tensors");
            for (int i = stage_t0[s]; i < stage_t1[s]; ++i)
                CDP_REQUIRE(tens[i].stage == s + 1, "ZeRO-CDP frames: stages must be contiguous tensor ranges");
            framePp[s & 1] = std::max<int64_t>(framePp[s & 1], stage_hi[s] - stage_lo[s]);
        }
        for (auto &f : framePp) f = (f + 63) / 64 * 64;
        th_stride = framePp[0] + framePp[1];
        // the initial state (theta | zeros) in mapped pinned host memory: read by the step-1 state loads only
        CDP_CUDA(cudaHostAlloc(&init_host, size_t(P) * 8, cudaHostAllocMapped));
        std::memset(init_host, 0, size_t(P) * 8);
        void *d = nullptr;
        CDP_CUDA(cudaHostGetDevicePointer(&d, init_host, 0));
        init_dev = static_cast<const float *>(d);
        for (size_t i = 0; i < tens.size(); ++i) {
            const int s = tens[i].stage - 1;
            foff[i] = (s & 1 ? framePp[0] : 0) + (tens[i].base - stage_lo[s]);
        }
    }
    // GEMM compute copies: per tensor (full replica) or per frame with stage-relative sub-buffers.
    void alloc_compute_copies() {
        for (int v = 0; v < 2; ++v) {
            wcv[v].assign(tens.size(), CTensor{});
            if (!frames) {
                for (auto &ts : tens) wc[v].push_back(ts.kind == T_BN ? CBuf{} : make_cbuf(kind, ts.rows, ts.cols));
                for (size_t i = 0; i < tens.size(); ++i) wcv[v][i] = wc[v][i].view();
                continue;
            }
            const size_t esz = kind == 0 ? 2 : 4;
            std::vector<size_t> off(tens.size(), 0);
            size_t frame_bytes[2] = {0, 0};  // per frame parity: the largest stage's compute copies
            for (size_t s = 0; s < stage_t0.size(); ++s) {
                size_t o = 0;
                for (int i = stage_t0[s]; i < stage_t1[s]; ++i) {
                    if (tens[i].kind == T_BN) continue;
                    off[i] = o;
                    o += (size_t(tens[i].rows) * round_up(std::max(tens[i].cols, 1), 16) * esz + 255) / 256 * 256;
                }
                frame_bytes[s & 1] = std::max(frame_bytes[s & 1], o);
            }
            wcpool[v][0] = DevBuf(frame_bytes[0] + frame_bytes[1]);
            if (kind == 1) wcpool[v][1] = DevBuf(frame_bytes[0] + frame_bytes[1]);
            for (size_t i = 0; i < tens.size(); ++i) {
                if (tens[i].kind == T_BN) continue;
                const size_t o = ((tens[i].stage - 1) & 1 ? frame_bytes[0] : 0) + off[i];
                wcv[v][i] = CTensor{wcpool[v][0].as<uint8_t>() + o,
                                    kind == 1 ? static_cast<void *>(wcpool[v][1].as<uint8_t>() + o) : nullptr,
                                    round_up(std::max(tens[i].cols, 1), 16)};
            }
        }
    }
    float *thp(int slot, int tensor) const { return theta[slot] + foff[tensor]; }
    // a "virtual base" whose element tens[tensor].base lands on the tensor's first value (kernels index by base)
    float *thv(int slot, int tensor) const { return theta[slot] + foff[tensor] - tens[tensor].base; }
    float *velv(int tensor) const { return vel ? vel + foff[tensor] - tens[tensor].base : nullptr; }

    void build(const int *widths, const int *depths, int n_layers) {
        int H = Hin, W = Win;
        // stem
        if (stem_kind == 0) {
            stem = add_conv(Cin0, widths[0], 3, 1, H, W, -1);
            stem_act = add_act(H, W, widths[0]);
        } else {
            stem = add_conv(Cin0, widths[0], 7, 2, H, W, -1);
            convs[stem].pad = 3;
            H = convs[stem].Ho;
            W = convs[stem].Wo;
            stem_act = add_act(H, W, widths[0]);
            H = (H + 2 - 3) / 2 + 1;
            W = (W + 2 - 3) / 2 + 1;
            pool_act = add_act(H, W, widths[0]);
        }
        int a = pool_act >= 0 ? pool_act : stem_act;
        int cin = widths[0];
        const int expansion = block_kind == 1 ? 4 : 1;
        for (int l = 0; l < n_layers; ++l) {
            for (int d = 0; d < depths[l]; ++d) {
                const int stride = (l > 0 && d == 0) ? 2 : 1;
                const int w = widths[l], cout = w * expansion;
                BlockL b;
                b.a_in = a;
                if (block_kind == 0) {
                    const int c1 = add_conv(cin, w, 3, stride, H, W, a);
                    const int Ho = convs[c1].Ho, Wo = convs[c1].Wo;
                    const int m = add_act(Ho, Wo, w);
                    const int c2 = add_conv(w, w, 3, 1, Ho, Wo, m);
                    b.convs = {c1, c2};
                    b.mid = {m};
                } else {
                    const int c1 = add_conv(cin, w, 1, 1, H, W, a);
                    const int m1 = add_act(H, W, w);
                    const int c2 = add_conv(w, w, 3, stride, H, W, m1);
                    const int Ho = convs[c2].Ho, Wo = convs[c2].Wo;
                    const int m2 = add_act(Ho, Wo, w);
                    const int c3 = add_conv(w, cout, 1, 1, Ho, Wo, m2);
                    b.convs = {c1, c2, c3};
                    b.mid = {m1, m2};
                }
                if (stride != 1 || cin != cout) b.ds = add_conv(cin, cout, 1, stride, H, W, a);
                const ConvL &last = convs[b.convs.back()];
                H = last.Ho;
                W = last.Wo;
                b.a_out = add_act(H, W, cout);
                blocks.push_back(b);
                a = b.a_out;
                cin = cout;
            }
        }
        fc_in = cin;
        fc_t = add_tensor(T_FC, int64_t(cin + 1) * classes, cin + 1, classes);
        P = tens.back().base + tens.back().n;
        if (stage_in)
            for (size_t i = 0; i < tens.size(); ++i) tens[i].stage = stage_in[i];
        // ---- buffers
        int64_t max_stats = 1, max_part = 1;
        for (auto &c : convs) {
            c.y = DevBuf(size_t(c.P) * c.cout * (kind == 0 ? 2 : 4));
            c.mean = DevBuf(c.cout * 4);
            c.rstd = DevBuf(c.cout * 4);
            c.dbeta = DevBuf(c.cout * 4);
            c.dgamma = DevBuf(c.cout * 4);
            c.dy = make_cbuf(kind, int(c.P), c.cout);
            max_stats = std::max<int64_t>(max_stats, int64_t(std::max(4 * c.tiles_fwd, 320)) * c.cout * 2);
            max_part = std::max<int64_t>(max_part, ((c.P + kBnRowsMin - 1) / kBnRowsMin) * c.cout * 2);
        }
        const ConvL &c0 = convs[stem];
        cols = make_cbuf(kind, int(c0.P), c0.K);
        for (auto &g : gbuf) g = DevBuf(size_t(max_act) * ysz());
        stats_fwd = DevBuf(size_t(max_stats) * 4);
        bnpart[0] = DevBuf(size_t(max_part) * 8);
        bnpart[1] = DevBuf(size_t(max_part) * 8);
        if (pool_act >= 0) pool_arg = DevBuf(size_t(act_P[pool_act]) * act_C[pool_act]);
        pooled = make_cbuf(kind, B, fc_in + 1);
        dz = make_cbuf(kind, B, classes);
        dpooled = DevBuf(size_t(B) * fc_in * 4);
        z = DevBuf(size_t(B) * classes * 4);
        loss_dev = DevBuf(8);
        loss_rows = DevBuf(size_t(B) * 8);
        region_off = (sizeof(RingFlags) + 255) / 256 * 256;
        Pp = (P + 63) / 64 * 64;
        layout_state();
        // shared region: RingFlags | theta slot 0 | theta slot 1 | partial | momentum (a slot is the full
        // parameter vector, or two stage frames in ZeRO-CDP mode)
        region = DevBuf(region_off + size_t(2 * th_stride + Pp + (momentum != 0.f ? th_stride : 0)) * 4);
        ring = region.as<RingFlags>();
        theta[0] = reinterpret_cast<float *>(region.as<uint8_t>() + region_off);
        theta[1] = theta[0] + th_stride;
        partial = theta[1] + th_stride;
        if (momentum != 0.f) vel = partial + Pp;
        cta_counters = DevBuf(2 * kMaxStages * 4);
        alloc_compute_copies();
        CDP_REQUIRE(int(tens.size()) <= kMaxStages, "too many parameter tensors for the ring flags");
        CDP_CUDA(cudaStreamCreateWithFlags(&main, cudaStreamNonBlocking));
        CDP_CUDA(cudaStreamCreateWithFlags(&cs, cudaStreamNonBlocking));
        CDP_CUDA(cudaStreamCreateWithFlags(&hs, cudaStreamNonBlocking));
        CDP_CUDA(cudaStreamCreateWithFlags(&ps, cudaStreamNonBlocking));
        ctrl_dev = DevBuf(sizeof(Control));
        perm_dev = DevBuf(size_t(B) * 4);
        flags_dev = DevBuf(sizeof(Flags));
        hist_loss = DevBuf(size_t(hist_cap) * 8);
        hist_flags = DevBuf(size_t(hist_cap) * sizeof(Flags));
        stage_bytes = (sizeof(Control) + size_t(B) * 4 + 255) / 256 * 256;
        CDP_CUDA(cudaMallocHost(&stage_host, stage_bytes * RING_N));
        for (auto &e : stage_ev) CDP_CUDA(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
        cnt_c = DevBuf(1 << 18);
        cnt_h = DevBuf(1 << 18);
        // split-K workspaces: a dry run of the step records the largest need per stream
        sizing = true;
        if (kind == 0)
            record_step<0>(0);
        else
            record_step<1>(0);
        sizing = false;
        for (auto e : events) cudaEventDestroy(e);
        events.clear();
        ws_c = DevBuf(std::max<size_t>(ws_c_floats, 1) * 4);
        ws_h = DevBuf(std::max<size_t>(ws_h_floats, 1) * 4);
    }

    // Algorithmic HBM bytes of the next GEMM launch (operands once, outputs, fused epilogue
    // operands / optimizer state): set by the caller, consumed by run_plan / run_pk (the bench's
    // roofline picks HBM or tensor per class from flops / bytes).
    double gemm_bytes = 0.0;
    double take_bytes() {
        const double b = gemm_bytes;
        gemm_bytes = 0.0;
        return b;
    }
    // per-parameter optimizer-state bytes of a hop / update epilogue
    double hop_bytes_per_param() const {
        const double wc_b = kind == 0 ? 2.0 : 8.0;
        if (world == 1) return 16.0 + wc_b + (vel ? 0.0 : -8.0);  // G = g: theta, v read + written, compute copy
        if (rank == 0) return 4.0;                                  // S = g
        if (rank < world - 1) return 8.0;                           // S = S_in + g
        return 20.0 + wc_b + (vel ? 0.0 : -8.0);                    // S_in + update
    }

    // ---------------------------------------------------------------- GEMM plumbing
    int splits_for(int64_t tiles, int64_t kblocks) const {
        const int nseg = kind == 0 ? 1 : 3;
        const int64_t total = kblocks * nseg;
        int64_t s = std::max<int64_t>(1, (2 * 148 + tiles - 1) / tiles);
        s = std::min(s, total);
        const int64_t per = (total + s - 1) / s;
        return int((total + per - 1) / per);
    }
    float *ws_for(bool hop) {
        if (sizing) return reinterpret_cast<float *>(uintptr_t(256));  // placeholder: plans only, no launch
        return hop ? ws_h.as<float>() : ws_c.as<float>();
    }
    int *cnt_for(bool hop) { return hop ? cnt_h.as<int>() : cnt_c.as<int>(); }

    // Account for / check the split-K workspace of a plan, then launch it.
    template <int K, int BN, bool AMN, bool BMN, class Epi, int MODE>
    void run_plan(const char *name, double flops, const GemmPlan &p, const typename Epi::Params &ep, cudaStream_t s,
                  bool hop) {
        const size_t need = gemm_ws_floats(p, BN);
        size_t &cap = hop ? ws_h_floats : ws_c_floats;
        if (sizing) {
            cap = std::max(cap, need);
            return;
        }
        CDP_REQUIRE(need <= cap, "split-K workspace too small");
        CDP_REQUIRE(size_t(p.grid.x) * p.grid.y * 4 <= (1u << 18), "split-K counters too small");
        L(name, flops, take_bytes(), s, [&] { launch_gemm<K, BN, AMN, BMN, Epi, MODE>(p, ep, s); });
    }

    static Operand opnd(const CTensor &t, bool lo, bool mn, int64_t mn_ext, int64_t k_ext) {
        return Operand{lo ? t.lo : t.hi, mn, uint64_t(mn_ext), uint64_t(k_ext), uint64_t(t.ld)};
    }

    // Plain GEMM D[M,N] = A.B (3 segments in the 3xTF32 mode).
    template <int K, bool AMN, bool BMN, class Epi>
    void gemm(const char *name, int BN, const CTensor &a, const CTensor &b, int64_t M, int64_t N, int64_t Kd,
              const typename Epi::Params &ep, cudaStream_t s, bool hop) {
        Operand A[3], Bo[3];
        int nseg = 1;
        A[0] = opnd(a, false, AMN, M, Kd);
        Bo[0] = opnd(b, false, BMN, N, Kd);
        if (K == 1) {
            nseg = 3;
            A[1] = A[0];
            Bo[1] = opnd(b, true, BMN, N, Kd);
            A[2] = opnd(a, true, AMN, M, Kd);
            Bo[2] = Bo[0];
        }
        const int bk = K == 0 ? 64 : 32;
        const int64_t tiles = ((M + 127) / 128) * ((N + BN - 1) / BN);
        const int splits = splits_for(tiles, (Kd + bk - 1) / bk);
        bn_switch(BN, [&](auto bnc) {
            constexpr int BNc = decltype(bnc)::value;
            if constexpr ((!BMN || BNc % (K == 0 ? 64 : 32) == 0) && (!Epi::kTile || BNc <= 64)) {
                GemmPlan p = plan_gemm<K, BNc, AMN, BMN>(A, Bo, nseg, int(M), int(N), int(Kd), splits, ws_for(hop),
                                                          cnt_for(hop));
                run_plan<K, BNc, AMN, BMN, Epi, GM_PLAIN>(name, 2.0 * M * N * Kd, p, ep, s, hop);
            } else {
                throw CdpError("unsupported GEMM configuration");
            }
        });
    }

    Nhwc nhwc_act(int a) const {
        const CBuf &t = acts[a];
        return Nhwc{t.hi.p, t.lo.p, t.ld, act_C[a], act_W[a], act_H[a], B};
    }
    Nhwc nhwc_dy(const ConvL &c) const { return Nhwc{c.dy.hi.p, c.dy.lo.p, c.dy.ld, c.cout, c.Wo, c.Ho, B}; }

    // ---------------------------------------------------------------- persistent GEMM path
    int sms_ = 0;
    int last_stat_slots = 0, last_grid = 0;
    bool last_fused = false;
    int sms() {
        if (!sms_) sms_ = num_sms();
        return sms_;
    }

    // phases / nph > 1: a stride-2 data gradient with its sub-pixel phases as one launch (the unit's
    // batch index is its phase; no split-K)
    template <int K, int BNc, bool AMN, bool BMN, class Epi, int MODE>
    void run_pk(const char *name, double flops, const GemmPlan &gp, const typename Epi::Params &ep_in, cudaStream_t s,
                bool hop, const ConvGeom *phases = nullptr, int nph = 1) {
        PkArgs a{};
        a.M = gp.args.M;
        a.N = gp.args.N;
        a.tiles_m = int(gp.grid.x);
        a.tiles_n = int(gp.grid.y);
        a.kb_per_seg = gp.args.kb_per_seg;
        a.n_seg = gp.args.n_seg;
        a.total_iters = a.kb_per_seg * a.n_seg;
        a.nph = nph;
        if (nph > 1) {
            a.nbatch = nph;
            for (int i = 0; i < nph; ++i) a.cvp[i] = phases[i];
            int mx = 0;
            for (int i = 0; i < nph; ++i) mx = std::max(mx, phases[i].ntap * phases[i].cpt * a.n_seg);
            a.total_iters = mx;
        }
        const int tiles = a.tiles_m * a.tiles_n * nph;
        int splits = 1;
        if (tiles < sms() && nph == 1 && !pk_direct<Epi>::value)
            splits = std::max(1, std::min(sms() / tiles, a.total_iters / split_min_kb()));  // units <= one wave
        a.iters_per_split = (a.total_iters + splits - 1) / splits;
        if (K == 1 && nph == 1) {
            // fp32 mode: the TMEM accumulator is not exact fp32 over long K, and the small 3xTF32 cross
            // terms must not be summed into the large hi.hi accumulation: every unit covers at most 256
            // of K inside ONE segment (a divisor of the segment's k-blocks); pk_reduce_kernel then sums
            // the partials in fp32 in split order (tests/test_gpu_gemm.py).  Plain GEMMs (1x1 convs, the
            // stem) were the fp32 path's main error: update rel-L2 2.4e-3 -> 2.8e-6 on the bottleneck
            // case.  (Merged stride-2 phases stay unsplit: their partials would share the workspace.)
            int ips = std::min(a.iters_per_split, std::min(a.kb_per_seg, 8));
            while (a.kb_per_seg % ips) --ips;
            a.iters_per_split = ips;
        }
        a.splits = (a.total_iters + a.iters_per_split - 1) / a.iters_per_split;
        using PL = PkLaunch<K, BNc, AMN, BMN, Epi, MODE>;
        a.units = tiles * a.splits;
        last_fused = a.splits == 1;
        const int slots_per_tile = 4;  // BN statistics slots per split tile: one per 32-row reduce chunk
        typename Epi::Params ep = a.splits > 1 ? Epi::for_split(ep_in) : ep_in;
        if constexpr (std::is_same<Epi, EpiConvOut2<K>>::value)
            if (a.splits > 1) ep.tiles = a.tiles_m * slots_per_tile;
        a.boxed = (MODE == GM_FPROP || MODE == GM_DGRAD) ? 1 : 0;
        a.cv = gp.args.cv;
        const size_t need = a.splits > 1 ? size_t(tiles) * a.splits * 128 * BNc : 0;
        size_t &cap = hop ? ws_h_floats : ws_c_floats;
        if (sizing) {
            cap = std::max(cap, need);
            return;
        }
        CDP_REQUIRE(need <= cap, "split-K workspace too small");
        a.ws = ws_for(hop);
        bool paired = false;
        const int grid = PL::prepare(a, sms(), paired);
        GemmMaps maps = gp.maps;
        PL::setup_tma_out(maps, a, ep);
        PL::setup_tma_add(maps, a, ep);
        // EpiConvOut2 statistics rows (grouped TMA-store epilogue: one slot per CTA and epilogue group)
        last_stat_slots = a.splits > 1 ? a.tiles_m * slots_per_tile : grid * (a.grouped ? 2 : 1);
        last_grid = grid;
        L(name, flops, take_bytes(), s, [&] { PL::launch(maps, a, ep, s, grid, paired); });
        if constexpr (!pk_direct<Epi>::value) if (a.splits > 1) {
            constexpr bool kStats = std::is_same<Epi, EpiConvOut2<K>>::value;
            constexpr int RC = kStats ? 32 : 16;  // rows per block: 256 threads x 2 float4 (stats) / 1 float4 (hop)
            constexpr int CC = 64;
            L("splitk_reduce", 0, double(need) * 4, s, [&] {
                launch_pdl(pk_reduce_kernel<BNc, Epi, RC, CC>, dim3(tiles, 128 / RC, BNc / CC), dim3(256), 0, s, a,
                           ep);
            });
        }
    }

    template <int K, bool AMN, bool BMN, class Epi>
    void pk_plain(const char *name, int BN, const CTensor &a, const CTensor &b, int64_t M, int64_t N, int64_t Kd,
                  const typename Epi::Params &ep, cudaStream_t s, bool hop) {
        Operand A[3], Bo[3];
        int nseg = 1;
        A[0] = opnd(a, false, AMN, M, Kd);
        Bo[0] = opnd(b, false, BMN, N, Kd);
        if (K == 1) {
            nseg = 3;
            A[1] = A[0];
            Bo[1] = opnd(b, true, BMN, N, Kd);
            A[2] = opnd(a, true, AMN, M, Kd);
            Bo[2] = Bo[0];
        }
        bn_switch(BN, [&](auto bnc) {
            constexpr int BNc = decltype(bnc)::value;
            if constexpr (BNc >= 64 && (!BMN || BNc % (K == 0 ? 64 : 32) == 0)) {
                GemmPlan p = plan_gemm<K, BNc, AMN, BMN>(A, Bo, nseg, int(M), int(N), int(Kd), 1, nullptr, nullptr);
                run_pk<K, BNc, AMN, BMN, Epi, GM_PLAIN>(name, 2.0 * M * N * Kd, p, ep, s, hop);
            } else {
                throw CdpError("unsupported GEMM configuration");
            }
        });
    }

    template <int K, int MODE, class Epi>
    void pk_conv(const char *name, int BN, const ConvL &c, const CTensor &w, const typename Epi::Params &ep,
                 cudaStream_t s, bool hop, int phase = -1) {
        const Nhwc a = c.in_act >= 0 ? nhwc_act(c.in_act) : Nhwc{};
        const Nhwc dy = nhwc_dy(c);
        double flops = 2.0 * double(c.P) * c.K * c.cout;
        if (phase >= 0) {  // one sub-pixel phase: its taps only
            ConvGeom probe{};
            dgrad_taps(probe, c.R, c.S, c.pad, phase);
            flops = 2.0 * double(c.P) * probe.ntap * c.cin * c.cout;
        }
        bn_switch(BN, [&](auto bnc) {
            constexpr int BNc = decltype(bnc)::value;
            constexpr bool AMN = MODE == GM_WGRAD, BMN = MODE != GM_DGRAD;
            if constexpr (BNc >= 64 && (!BMN || BNc % (K == 0 ? 64 : 32) == 0)) {
                GemmPlan p = plan_conv<K, BNc, MODE>(a, w.hi, w.lo, w.ld, dy, c.R, c.S, c.stride, c.pad, c.cin,
                                                     c.cout, 1, nullptr, nullptr, phase);
                run_pk<K, BNc, AMN, BMN, Epi, MODE>(name, flops, p, ep, s, hop);
            } else {
                throw CdpError("unsupported conv GEMM configuration");
            }
        });
    }

    // Stride-2 data gradient: the sub-pixel phases with taps as one launch (shared dy / W maps and
    // pixel boxes; per-phase tap tables and output offsets).
    template <int K, class Epi>
    void pk_dgrad_phases(const char *name, int BN, const ConvL &c, const CTensor &w, const typename Epi::Params &ep,
                         cudaStream_t s) {
        CDP_REQUIRE(c.in_act >= 0, "stride-2 data gradient of the stem is never needed");
        const Nhwc a = nhwc_act(c.in_act);
        const Nhwc dy = nhwc_dy(c);
        bn_switch(BN, [&](auto bnc) {
            constexpr int BNc = decltype(bnc)::value;
            if constexpr (BNc >= 64) {
                ConvGeom ph[4];
                GemmPlan first{};
                int nph = 0;
                double flops = 0.0;
                for (int phase = 0; phase < 4; ++phase) {
                    ConvGeom probe{};
                    dgrad_taps(probe, c.R, c.S, c.pad, phase);
                    if (probe.ntap == 0) continue;
                    GemmPlan p = plan_conv<K, BNc, GM_DGRAD>(a, w.hi, w.lo, w.ld, dy, c.R, c.S, c.stride,
                                                             c.pad, c.cin, c.cout, 1, nullptr, nullptr, phase);
                    if (nph == 0) first = p;
                    ph[nph++] = p.args.cv;
                    flops += 2.0 * double(c.P) * probe.ntap * c.cin * c.cout;
                }
                run_pk<K, BNc, false, false, Epi, GM_DGRAD>(name, flops, first, ep, s, false, ph, nph);
            } else {
                throw CdpError("unsupported conv GEMM configuration");
            }
        });
    }

    static int blocks_for(int64_t n, int per = 256) { return int(std::min<int64_t>(8 * 148, (n + per - 1) / per)); }
    // grid-stride elementwise kernels: at most one wave of resident 256-thread CTAs (blocks_for's 8 per SM is
    // two waves for a kernel that holds 4; CDP_BN_GRID_OCC=0 keeps blocks_for)
    template <class Kern>
    int resident_blocks(Kern kern, int64_t n) {
        static const int64_t max_vec = [] {  // vectors (8 elements) up to which the one-wave grid is used
            const char *e = std::getenv("CDP_BN_GRID_OCC");
            return e ? std::atoll(e) : (int64_t(1) << 20);
        }();
        if (n > max_vec) return blocks_for(n);
        int occ = 0;
        CDP_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, kern, 256, 0));
        return int(std::min<int64_t>(int64_t(std::max(occ, 1)) * sms(), (n + 255) / 256));
    }
    static int tile_n(int n) { return n <= 64 ? 64 : n <= 128 ? 128 : 256; }  // a supported BN covering n
    // tile-width probe (development): env `name` caps the GEMM tile width of one class
    static int tile_cap(const char *name, int bn) {
        const char *e = std::getenv(name);
        return e ? std::min(bn, std::atoi(e)) : bn;
    }

    // ---------------------------------------------------------------- forward pieces
    template <int K>
    void conv_forward(int ci, int vslot, cudaStream_t s) {
        ConvL &c = convs[ci];
        typename EpiConvOut2<K>::Params ep{};
        ep.out = c.y.p;
        ep.ld = c.cout;
        ep.stats = stats_fwd.as<float>();
        ep.tiles = c.tiles_fwd;
        const CTensor w = wcv[vslot][c.tw];
        rec(c.tw, A_FWD, 0, vslot, s);
        gemm_bytes = double(c.impl == CI_STEM ? c.P * cols.ld : c.Pin * c.cin) * esz() +
                     double(c.K) * c.cout * esz() + double(c.P) * c.cout * ysz();
        if (c.impl == CI_IMPLICIT) {
            pk_conv<K, GM_FPROP, EpiConvOut2<K>>("conv_fprop", tile_cap("CDP_PROBE_BN_FPROP3", tile_n(c.cout)), c, w,
                                                 ep, s, false);
        } else {
            const CTensor in = c.impl == CI_STEM ? cols.view() : acts[c.in_act].view();
            const int64_t Kd = c.impl == CI_STEM ? c.K : c.cin;
            // 1x1 forward with BN statistics: 128-column tiles (tensor-core statistics, better balance than 256:
            // measured 1.77 -> 1.59 ms per ResNet-50 step before the statistics MMAs)
            const int bnt = c.impl == CI_STEM ? tile_n(c.cout) : tile_cap("CDP_PROBE_FWD1X1_BN", std::min(tile_n(c.cout), 128));
            pk_plain<K, false, true, EpiConvOut2<K>>(c.impl == CI_STEM ? "stem_fprop" : "conv_fprop_1x1",
                                                     bnt, in, w, c.P, c.cout, Kd, ep, s, false);
        }
        rec(c.tw, A_FWD, 1, vslot, s);
        const int slots = sizing ? c.tiles_fwd : last_stat_slots;
        L("bn_finalize_fwd", 0, double(slots) * c.cout * 8, s, [&] {
            launch_pdl(bn_finalize_fwd_kernel, dim3((c.cout * 32 + 255) / 256), dim3(256), 0, s,
                       (const float *)stats_fwd.as<float>(), slots, c.cout, c.P, eps, c.mean.as<float>(),
                       c.rstd.as<float>());
        });
    }

    const float *gamma(int ci, int vslot) const { return thp(vslot, convs[ci].tb); }
    const float *beta(int ci, int vslot) const { return thp(vslot, convs[ci].tb) + convs[ci].cout; }
    int vs(int tensor, int p) const { return tens[tensor].fresh ? p : (p ^ 1); }
    // trace mode: one access record of `tensor`'s parameters in theta slot `slot` (stream order)
    void rec(int tensor, int akind, int phase, int slot, cudaStream_t s) {
        if (!trace) return;
        L("trace_record", 0, 0, s, [&] {
            access_record_kernel<<<1, 1, 0, s>>>(TraceLog{tlog.as<uint32_t>(), tcur.as<uint32_t>(), kTraceCap}, ring,
                                                 rank, tensor + 1, akind, phase, slot,
                                                 (const int *)&ctrl_dev.as<Control>()->step);
            CDP_CUDA(cudaGetLastError());
        });
    }
    // trace mode, around an update of `tensor` at step t (slot p): reads theta_t from p, writes t + 1 to p ^ 1
    template <class F>
    void traced_update(int tensor, int p, bool updates, cudaStream_t s, F &&launch) {
        if (updates) rec(tensor, A_UPD, 0, p, s);
        launch();
        if (trace && updates) {
            L("trace_vtag", 0, 0, s, [&] {
                vtag_update_kernel<<<1, 1, 0, s>>>(ring, tensor + 1, (const int *)&ctrl_dev.as<Control>()->step);
                CDP_CUDA(cudaGetLastError());
            });
            rec(tensor, A_NEW, 1, p ^ 1, s);
        }
    }
    int esz() const { return kind == 0 ? 2 : 8; }   // compute-format bytes per element
    int ysz() const { return kind == 0 ? 2 : 4; }   // Y-format (conv outputs, gradients) bytes per element

    template <int K>
    void bn_apply(int ci, int vslot, const BnResidual &res, const CTensor &out, cudaStream_t s, int res_ci = -1,
                  int res_slot = 0) {
        ConvL &c = convs[ci];
        rec(c.tb, A_FWD, 0, vslot, s);
        if (res_ci >= 0) rec(convs[res_ci].tb, A_FWD, 0, res_slot, s);
        const double bytes = double(c.P) * c.cout * (ysz() + esz() + (res.act.hi ? esz() : res.y ? ysz() : 0));
        L("bn_apply", 0, bytes, s, [&] {
            auto kern = res.act.hi ? bn_apply_kernel<K, 1> : res.y ? bn_apply_kernel<K, 2> : bn_apply_kernel<K, 0>;
            launch_pdl(kern, dim3(resident_blocks(kern, c.P * c.cout / 8)), dim3(256), 0, s, (const void *)c.y.p, c.P, c.cout,
                       (const float *)c.mean.as<float>(), (const float *)c.rstd.as<float>(), gamma(ci, vslot),
                       beta(ci, vslot), res, 1, out);
        });
        rec(c.tb, A_FWD, 1, vslot, s);
        if (res_ci >= 0) rec(convs[res_ci].tb, A_FWD, 1, res_slot, s);
    }

    template <int K>
    void forward(int p, cudaStream_t s, const std::function<void(int)> &pull) {
        ConvL &c0 = convs[stem];
        L("stem_im2col", 0, double(c0.P) * cols.ld * esz(), s, [&] {
            const size_t smem = size_t(c0.R) * (Win + 2 * c0.pad) * Cin0 * 4 + size_t(cols.ld) * 4;
            CDP_REQUIRE(smem <= 48 * 1024, "stem input rows exceed the shared-memory stage");
            CDP_REQUIRE((Win * Cin0) % 4 == 0, "stem rows are staged as 16-byte vectors (W * C % 4 == 0)");
            if (c0.R == 3)
                launch_pdl(stem_im2col_rows_kernel<K, 3, 3>, dim3(B * c0.Ho), dim3(256), smem, s,
                           (const float *)data_x.as<float>(), (const int *)perm_dev.as<int>(), Hin, Win, c0.stride,
                           c0.pad, c0.Ho, c0.Wo, cols.view());
            else
                launch_pdl(stem_im2col_rows_kernel<K, 7, 3>, dim3(B * c0.Ho), dim3(256), smem, s,
                           (const float *)data_x.as<float>(), (const int *)perm_dev.as<int>(), Hin, Win, c0.stride,
                           c0.pad, c0.Ho, c0.Wo, cols.view());
        });
        pull(c0.tw);
        pull(c0.tb);
        conv_forward<K>(stem, vs(c0.tw, p), s);
        zdone(c0.tw, 0, s);
        bn_apply<K>(stem, vs(c0.tb, p), BnResidual{}, acts[stem_act].view(), s);
        zdone(c0.tb, 0, s);
        if (pool_act >= 0) {
            const int a = stem_act, o = pool_act;
            L("maxpool_fwd", 0, double(act_P[a] + act_P[o]) * act_C[a] * esz(), s, [&] {
                launch_pdl(maxpool_fwd_kernel<K>, dim3(blocks_for(act_P[o] * act_C[o] / 8)), dim3(256), 0, s,
                           acts[a].view(), B, act_H[a], act_W[a], act_C[a], act_H[o], act_W[o], acts[o].view(),
                           pool_arg.as<uint8_t>());
            });
        }
        for (auto &b : blocks) {
            const int n = int(b.convs.size());
            for (int i = 0; i < n; ++i) {
                ConvL &c = convs[b.convs[i]];
                pull(c.tw);
                pull(c.tb);
                conv_forward<K>(b.convs[i], vs(c.tw, p), s);
                zdone(c.tw, 0, s);
                if (i < n - 1) {
                    bn_apply<K>(b.convs[i], vs(c.tb, p), BnResidual{}, acts[b.mid[i]].view(), s);
                    zdone(c.tb, 0, s);
                }
            }
            BnResidual res{};
            if (b.ds >= 0) {
                ConvL &cd = convs[b.ds];
                pull(cd.tw);
                pull(cd.tb);
                conv_forward<K>(b.ds, vs(cd.tw, p), s);
                zdone(cd.tw, 0, s);
                res.y = cd.y.p;
                res.mean = cd.mean.as<float>();
                res.rstd = cd.rstd.as<float>();
                res.gamma = gamma(b.ds, vs(cd.tb, p));
                res.beta = beta(b.ds, vs(cd.tb, p));
            } else {
                res.act = acts[b.a_in].view();
            }
            const int last = b.convs.back();
            bn_apply<K>(last, vs(convs[last].tb, p), res, acts[b.a_out].view(), s, b.ds,
                        b.ds >= 0 ? vs(convs[b.ds].tb, p) : 0);
            zdone(convs[last].tb, 0, s);
            if (b.ds >= 0) zdone(convs[b.ds].tb, 0, s);
        }
        // pool + classifier
        const int la = blocks.empty() ? stem_act : blocks.back().a_out;
        const int HW = int(act_P[la] / B);
        L("avgpool", 0, double(act_P[la]) * fc_in * esz(), s, [&] {
            launch_pdl(avgpool_kernel<K>, dim3(B), dim3(256), 0, s, acts[la].view(), B, HW, fc_in, pooled.view());
        });
        pull(fc_t);
        typename EpiFwd<K>::Params ep{};
        ep.last = 1;
        ep.z = z.as<float>();
        rec(fc_t, A_FWD, 0, vs(fc_t, p), s);
        gemm<K, true, false, EpiFwd<K>>("fc_fwd", 32, wcv[vs(fc_t, p)][fc_t], pooled.view(), classes, B,
                                        fc_in + 1, ep, s, false);
        rec(fc_t, A_FWD, 1, vs(fc_t, p), s);
        zdone(fc_t, 0, s);
    }

    // ---------------------------------------------------------------- backward pieces
    // BN backward of conv ci (and of the projection conv `ds` sharing g' and the mask):
    // statistics, finalise, dy = BN'(g') in compute format.
    template <int K>
    void bn_backward(int ci, int ds, int p, const void *g, const CTensor &mask, cudaStream_t s) {
        ConvL &c = convs[ci];
        zrecv<K>(c.tb, 1, s);
        if (ds >= 0) zrecv<K>(convs[ds].tb, 1, s);
        static const bool stats4 = std::getenv("CDP_BN_STATS4") != nullptr;  // A/B: the 4-channel kernel
        const bool s8 = K == 0 && c.cout % 8 == 0 && !stats4;
        const int rows_blk = bn_rows_per_block(c.P, c.cout);  // kBnRowsMin or kBnRows
        int nblk = int((c.P + rows_blk - 1) / rows_blk);
        const int C4 = c.cout / 4, TPR = C4 < 32 ? C4 : 32;
        const ConvL *cd = ds >= 0 ? &convs[ds] : nullptr;
        const double bytes = double(c.P) * c.cout * (ysz() + (mask.hi ? esz() : 0) + ysz() + (cd ? ysz() : 0));
        if (s8) {
            const int C8 = c.cout / 8, T8 = C8 < 32 ? C8 : 32, gy = (C8 + T8 - 1) / T8;
            const int64_t chunk = int64_t(256 / T8) * (cd ? 2 : 4);
            const int64_t nchunks = (c.P + chunk - 1) / chunk;
            // two CTAs per SM over the channel groups, at most one chunk per CTA, within the partial buffer
            nblk = int(std::min<int64_t>({nchunks, std::max(1, 2 * sms() / gy), (c.P + kBnRowsMin - 1) / kBnRowsMin}));
            L("bn_bwd_stats", 0, bytes, s, [&] {
                auto kern = mask.hi ? (cd ? bn_bwd_stats8_kernel<true, true> : bn_bwd_stats8_kernel<true, false>)
                                    : (cd ? bn_bwd_stats8_kernel<false, true> : bn_bwd_stats8_kernel<false, false>);
                launch_pdl(kern, dim3(nblk, gy), dim3(256), 0, s,
                           (const __nv_bfloat16 *)g, (const __nv_bfloat16 *)mask.hi, c.P, c.cout,
                           (const __nv_bfloat16 *)c.y.p, (const float *)c.mean.as<float>(),
                           (const float *)c.rstd.as<float>(), bnpart[0].as<double>(),
                           cd ? (const __nv_bfloat16 *)cd->y.p : (const __nv_bfloat16 *)nullptr,
                           cd ? (const float *)cd->mean.as<float>() : (const float *)nullptr,
                           cd ? (const float *)cd->rstd.as<float>() : (const float *)nullptr,
                           cd ? bnpart[1].as<double>() : (double *)nullptr);
            });
        } else
        L("bn_bwd_stats", 0, bytes, s, [&] {
            auto kern = rows_blk == kBnRowsMin ? bn_bwd_stats_kernel<K, kBnRowsMin>
                        : rows_blk == kBnRows  ? bn_bwd_stats_kernel<K, kBnRows>
                                               : bn_bwd_stats_kernel<K, kBnRowsBig>;
            launch_pdl(kern, dim3(nblk, (C4 + TPR - 1) / TPR), dim3(256), 0, s, g, mask, c.P,
                       c.cout, (const void *)c.y.p, (const float *)c.mean.as<float>(),
                       (const float *)c.rstd.as<float>(), bnpart[0].as<double>(),
                       cd ? (const void *)cd->y.p : (const void *)nullptr,
                       cd ? (const float *)cd->mean.as<float>() : (const float *)nullptr,
                       cd ? (const float *)cd->rstd.as<float>() : (const float *)nullptr,
                       cd ? bnpart[1].as<double>() : (double *)nullptr);
        });
        for (int k = 0; k < (cd ? 2 : 1); ++k) {
            ConvL &cc = k == 0 ? c : convs[ds];
            L("bn_finalize_bwd", 0, double(nblk) * cc.cout * 16, s, [&] {
                launch_pdl(bn_finalize_bwd_kernel, dim3((cc.cout * 32 + 255) / 256), dim3(256), 0, s,
                           (const double *)bnpart[k].as<double>(), nblk, cc.cout, cc.dbeta.as<float>(),
                           cc.dgamma.as<float>());
            });
            bn_bwd_apply<K>(k == 0 ? ci : ds, p, g, mask, s);
        }
    }

    template <int K>
    void bn_bwd_apply(int ci, int p, const void *g, const CTensor &mask, cudaStream_t s) {
        ConvL &cc = convs[ci];
        const int vslot = vs(cc.tb, p);
        rec(cc.tb, A_BWD, 0, vslot, s);
        L("bn_bwd_apply", 0, double(cc.P) * cc.cout * (2 * ysz() + (mask.hi ? 2 : 1) * esz()), s, [&] {
            auto kern = mask.hi ? bn_bwd_apply_kernel<K, true> : bn_bwd_apply_kernel<K, false>;
            launch_pdl(kern, dim3(resident_blocks(kern, cc.P * cc.cout / 8)), dim3(256), 0, s, g, mask,
                       (const void *)cc.y.p, cc.P, cc.cout, (const float *)cc.mean.as<float>(),
                       (const float *)cc.rstd.as<float>(), gamma(ci, vslot), (const float *)cc.dbeta.as<float>(),
                       (const float *)cc.dgamma.as<float>(), cc.dy.view());
        });
        rec(cc.tb, A_BWD, 1, vslot, s);
    }

    template <class P>
    static P ep_with(P ep, void *out, int ld) {
        ep.out = out;
        ep.ld = ld;
        return ep;
    }
    // the TMA-staged residual-add epilogue exists for bf16 (KIND 0) only
    template <int K, class F>
    static void pk_tadd(F &&f) {
        if constexpr (K == 0) f(EpiConvAddT<0>{});
    }
    // conv data gradient into g_in (fp32 [Pin][cin]).
    // add != null: g_in = dgrad + (add masked by add_mask) (the block's residual branch).
    template <int K>
    void conv_dgrad(int ci, int vslot, void *g_in, cudaStream_t s, const void *add = nullptr,
                    CTensor add_mask = CTensor{}, CTensor out_mask = CTensor{}) {
        ConvL &c = convs[ci];
        zrecv<K>(c.tw, 1, s);
        const CTensor w = wcv[vslot][c.tw];
        rec(c.tw, A_BWD, 0, vslot, s);
        typename EpiConvOut2<K>::Params ep{};
        ep.stats = nullptr;
        ep.add = add;
        ep.add_mask = add_mask;
        ep.out_mask = out_mask;
        gemm_bytes = double(c.P) * c.cout * esz() + double(c.K) * c.cout * esz() + double(c.Pin) * c.cin * ysz() +
                     (add ? double(c.Pin) * c.cin * ysz() : 0.0) +
                     double(c.Pin) * c.cin * esz() * ((add_mask.hi ? 1 : 0) + (out_mask.hi ? 1 : 0));
        // residual-gradient add: the direct (register) epilogue, its own GEMM instantiation
        const bool direct = EpiConvAdd<K>::eligible(ep_with(ep, g_in, c.cin), c.cin, tile_n(c.cin)) &&
                            std::getenv("CDP_NO_DIRECT_ADD") == nullptr;
        // residual / mask rows staged by TMA (tiles of 128 / 256 columns; CDP_NO_TMA_ADD=1 disables)
        static const bool tma_add_on = std::getenv("CDP_NO_TMA_ADD") == nullptr;
        const bool tadd = K == 0 && direct && tma_add_on && tile_n(c.cin) >= 128 && c.impl == CI_PLAIN;
        if (c.impl == CI_PLAIN) {
            ep.out = g_in;
            ep.ld = c.cin;
            if (tadd)
                pk_tadd<K>([&](auto e) {
                    pk_plain<K, false, false, decltype(e)>("conv_dgrad_1x1", tile_cap("CDP_PROBE_BN_DGRAD1", tile_n(c.cin)), c.dy.view(), w,
                                                           c.P, c.cin, c.cout, ep, s, false);
                });
            else if (direct)
                pk_plain<K, false, false, EpiConvAdd<K>>("conv_dgrad_1x1", tile_n(c.cin), c.dy.view(), w, c.P,
                                                         c.cin, c.cout, ep, s, false);
            else
                pk_plain<K, false, false, EpiConvOut2<K>>("conv_dgrad_1x1", tile_n(c.cin), c.dy.view(), w,
                                                          c.P, c.cin, c.cout, ep, s, false);
        } else if (c.stride == 1) {
            ep.out = g_in;
            ep.ld = c.cin;
            if (tadd)
                pk_tadd<K>([&](auto e) { pk_conv<K, GM_DGRAD, decltype(e)>("conv_dgrad", tile_n(c.cin), c, w, ep, s, false); });
            else if (direct)
                pk_conv<K, GM_DGRAD, EpiConvAdd<K>>("conv_dgrad", tile_n(c.cin), c, w, ep, s, false);
            else
                pk_conv<K, GM_DGRAD, EpiConvOut2<K>>("conv_dgrad", tile_n(c.cin), c, w, ep, s, false);
        } else {
            // stride 2: four sub-pixel phases, each a stride-1 implicit GEMM over dy with its own taps
            // (pixels (2i + ph, 2j + pw)); phases without taps (1x1 convs) leave zeros
            ep.out = g_in;
            ep.ld = c.cin;
            if (c.R == 1) {
                CDP_REQUIRE(add == nullptr, "a 1x1 stride-2 data gradient cannot fold a residual branch");
                if (!sizing) CDP_CUDA(cudaMemsetAsync(g_in, 0, size_t(c.Pin) * c.cin * ysz(), s));
            }
            pk_dgrad_phases<K, EpiConvOut2<K>>("conv_dgrad_s2", tile_n(c.cin), c, w, ep, s);
        }
        rec(c.tw, A_BWD, 1, vslot, s);
    }

    HopParams hop_params(int tensor, int p) {
        const TensorSpec &ts = tens[tensor];
        HopParams hp{};
        hp.mode = world == 1 ? 3 : (rank == 0 ? 0 : rank == world - 1 ? 2 : 1);
        hp.stage = tensor + 1;
        hp.base = ts.base;
        hp.din = ts.rows;
        hp.dout = ts.cols;
        hp.s_in = rank > 0 ? prev_partial : partial;
        hp.s_out = partial;
        hp.theta_cur = thv(p, tensor);
        hp.theta_new = thv(p ^ 1, tensor);
        hp.vel = velv(tensor);
        hp.lr = &ctrl_dev.as<Control>()->lr;
        hp.momentum = momentum;
        hp.wd = wd;
        hp.n_mb = float(world);
        hp.wc_new = ts.kind == T_BN ? CTensor{} : wcv[p ^ 1][tensor];
        Flags *fl = flags_dev.as<Flags>();
        hp.grad_flags = &fl->grad;
        hp.upd_flags = &fl->upd;
        hp.sync.enabled = 1;
        // ZeRO-CDP: no parameter pulls; pull chain: only the first reader takes from the updater
        hp.sync.n_readers = zero ? 0 : !chain.empty() ? 1 : world - 1;
        hp.sync.step = &ctrl_dev.as<Control>()->step;
        hp.sync.own = ring;
        hp.sync.prev = prev_ring;
        hp.sync.cta_counter = cta_counters.as<unsigned>();
        hp.sync.pre_external = 1;
        if (allreduce) {  // gradient of this rank's micro-batch only, into the flat buffer
            hp.mode = 4;
            hp.s_out = partial;
            hp.sync.enabled = 0;
        }
        return hp;
    }

    // DP all-reduce baseline: the update of the step just run from the summed flat gradient
    // (tensors [t0, t1): the ZeRO-DP baseline updates only the stage this rank owns).
    void apply_update(int t0 = 0, int t1 = -1) {
        CDP_REQUIRE(allreduce, "apply_update is the DP all-reduce baseline's update");
        CDP_REQUIRE(t >= 2, "no step has run");
        if (t1 < 0) t1 = int(tens.size());
        CDP_REQUIRE(t0 >= 0 && t0 <= t1 && t1 <= int(tens.size()), "tensor range out of bounds");
        const int p = (t - 1) & 1;
        Flags *fl = flags_dev.as<Flags>();
        for (size_t k = size_t(t0); k < size_t(t1); ++k) {
            const TensorSpec &ts = tens[k];
            HopParams hp{};
            hp.mode = 3;
            hp.stage = int(k) + 1;
            hp.base = ts.base;
            hp.s_in = partial;
            hp.theta_cur = thv(p, int(k));
            hp.theta_new = thv(p ^ 1, int(k));
            hp.vel = velv(int(k));
            hp.lr = &ctrl_dev.as<Control>()->lr;
            hp.momentum = momentum;
            hp.wd = wd;
            hp.n_mb = float(world);
            hp.wc_new = ts.kind == T_BN ? CTensor{} : wcv[p ^ 1][k];
            hp.upd_flags = &fl->upd;
            if (kind == 0)
                launch_pdl(update_flat_kernel<0>, dim3(blocks_for(ts.n)), dim3(256), 0, main, hp, ts.n,
                           std::max(ts.cols, 1));
            else
                launch_pdl(update_flat_kernel<1>, dim3(blocks_for(ts.n)), dim3(256), 0, main, hp, ts.n,
                           std::max(ts.cols, 1));
        }
    }

    // Ring waits of a hop (multi-GPU) ahead of its kernel on the hop stream.
    void hop_wait(const HopParams &hp, cudaStream_t s) {
        if (world == 1 || hp.mode >= 3) return;
        L("hop_wait", 0, 0, s, [&] { hop_wait_kernel<<<1, 128, 0, s>>>(hp); CDP_CUDA(cudaGetLastError()); });
    }

    // weight gradient of conv ci fused with its hop / update (hop stream).
    template <int K>
    void conv_wgrad_hop(int ci, int p, cudaStream_t s) {
        ConvL &c = convs[ci];
        HopParams hp = hop_params(c.tw, p);
        hop_wait(hp, s);
        traced_update(c.tw, p, hp.mode == 2 || hp.mode == 3, s, [&] {
            gemm_bytes = double(c.impl == CI_STEM ? c.P * cols.ld : c.Pin * c.cin) * esz() +
                         double(c.P) * c.cout * esz() + double(c.K) * c.cout * hop_bytes_per_param();
            if (c.impl == CI_IMPLICIT) {
                pk_conv<K, GM_WGRAD, EpiHop2<K>>("conv_wgrad_hop", tile_n(c.cout), c, wcv[0][c.tw], hp, s, true);
            } else {
                const CTensor in = c.impl == CI_STEM ? cols.view() : acts[c.in_act].view();
                pk_plain<K, true, true, EpiHop2<K>>(c.impl == CI_STEM ? "stem_wgrad_hop" : "conv_wgrad_hop_1x1",
                                                    tile_n(c.cout), in, c.dy.view(), c.K, c.cout, c.P, hp, s, true);
            }
        });
    }

    void bn_hop(int ci, int p, cudaStream_t s) {
        ConvL &c = convs[ci];
        HopParams hp = hop_params(c.tb, p);
        hop_wait(hp, s);
        traced_update(c.tb, p, hp.mode == 2 || hp.mode == 3, s, [&] {
            L("bn_hop", 0, double(c.cout) * 2 * 24, s, [&] {
                launch_pdl(vector_hop_kernel, dim3(1), dim3(128), 0, s, hp, (const float *)c.dgamma.as<float>(),
                           (const float *)c.dbeta.as<float>(), c.cout);
            });
        });
    }

    // ---------------------------------------------------------------- step capture
    cudaEvent_t ev(cudaStream_t s) {
        cudaEvent_t e;
        CDP_CUDA(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
        events.push_back(e);
        if (!sizing) CDP_CUDA(cudaEventRecord(e, s));
        return e;
    }
    void wait(cudaStream_t s, cudaEvent_t e) {
        if (!sizing) CDP_CUDA(cudaStreamWaitEvent(s, e, 0));
    }
    bool last_updater() const { return rank == world - 1; }

    // ---------------------------------------------------------------- ZeRO-CDP windows
    ZeroUse zuse(int tensor, int kindFB) const {
        const int st = tens[tensor].stage - 1;
        const int *e = &ztab[((size_t(st) * 2 + kindFB) * world + rank) * 3];
        return ZeroUse{e[0], e[1], e[2], 2 * world};
    }
    const float *peer_theta(int r, int slot) const {
        return reinterpret_cast<const float *>(peers[r] + region_off) + size_t(slot) * th_stride;
    }
    // Before this rank's first access to `tensor` in its F (0) / B (1) use: wait for the
    // predecessor, copy the state from its HBM.
    template <int K>
    void zrecv(int tensor, int kindFB, cudaStream_t s, int step_delta = 0, bool copy = true, bool auto_wait = true) {
        if (!zero || sizing) return;
        CDP_REQUIRE(int(peers.size()) == world, "ZeRO-CDP needs connected peers");
        const ZeroUse z = zuse(tensor, kindFB);
        // self-succession (the same rank's previous use of the stage): nothing to copy — except, with
        // frames, the step-1 load of the initial state (dstep -1: no predecessor in step 1)
        if (z.src == rank && !(frames && copy && z.dstep < 0)) return;
        const TensorSpec &ts = tens[tensor];
        const RingFlags *src_flags = reinterpret_cast<const RingFlags *>(peers[z.src]);
        if (frames && copy && z.src != rank && auto_wait) frame_wait(tens[tensor].stage, kindFB, s);
        if (z.src != rank) L("zero_wait", 0, 0, s, [&] {
            zero_wait_kernel<<<1, 32, 0, s>>>(z, rank, src_flags, ring, tensor + 1,
                                              (const int *)&ctrl_dev.as<Control>()->step, step_delta,
                                              (trace && copy) ? 1 : 0);
            CDP_CUDA(cudaGetLastError());
        });
        if (!copy) return;
        const float *sv =
            vel ? reinterpret_cast<const float *>(peers[z.src] + region_off) + 2 * th_stride + Pp + foff[tensor] : nullptr;
        CTensor w0 = ts.kind == T_BN ? CTensor{} : wcv[0][tensor];
        CTensor w1 = ts.kind == T_BN ? CTensor{} : wcv[1][tensor];
        if (z.src != rank) zero_bytes_per_step += ts.n * 4 * (vel ? 3 : 2);
        const float *it = frames ? init_dev + ts.base : nullptr;
        const float *iv = frames ? init_dev + P + ts.base : nullptr;
        L("zero_copy", 0, double(ts.n) * (vel ? 3 : 2) * 8, s, [&] {
            launch_pdl(zero_copy_kernel<K>, dim3(blocks_for(ts.n, 1024)), dim3(256), 0, s, z, rank,
                       peer_theta(z.src, 0) + foff[tensor], peer_theta(z.src, 1) + foff[tensor], sv, thp(0, tensor),
                       thp(1, tensor), vel ? vel + foff[tensor] : (float *)nullptr, ts.n, std::max(ts.cols, 1), w0,
                       w1, (const int *)&ctrl_dev.as<Control>()->step, it, iv);
        });
        if (frames && z.src != rank)
            L("zero_copied", 0, 0, s, [&] {
                zero_copied_kernel<<<1, 1, 0, s>>>(z, rank, reinterpret_cast<RingFlags *>(peers[z.src]), tensor + 1,
                                                   (const int *)&ctrl_dev.as<Control>()->step);
                CDP_CUDA(cudaGetLastError());
            });
    }
    // The frame-reuse wait of a window that starts with stage `stage`'s `kindFB` use on this rank (once
    // per window and recorded step: before its first state copy).
    void frame_wait(int stage, int kindFB, cudaStream_t s) {
        int &done = zwin_done[size_t(stage - 1) * 2 + kindFB];
        if (done) return;
        done = 1;
        const int N = world, per = 2 * N;
        // this rank's uses, three steps: (kind, stage, step offset) in order F1..FN, BN..B1
        struct Op {
            int k, st, dt;
        };
        std::vector<Op> ops;
        for (int dt = -3; dt <= 1; ++dt) {
            for (int j = 1; j <= N; ++j) ops.push_back({0, j, dt});
            for (int j = N; j >= 1; --j) ops.push_back({1, j, dt});
        }
        std::vector<std::pair<int, int>> win;  // [first op, last op]
        for (int i = 0; i < int(ops.size()); ++i) {
            if (!win.empty() && ops[win.back().second].st == ops[i].st)
                win.back().second = i;
            else
                win.push_back({i, i});
        }
        int w = -1;
        for (int i = 2; i < int(win.size()); ++i) {
            const Op &f = ops[win[i].first];
            if (f.k == kindFB && f.st == stage && f.dt == 0) w = i;
        }
        CDP_REQUIRE(w >= 2, "ZeRO-CDP frames: window not found");
        const Op &last = ops[win[w - 2].second];
        const int sp = last.st - 1;
        auto base_of = [&](int st0, int k, int r) { return ztab[((size_t(st0) * 2 + k) * world + r) * 3]; };
        const int bl = base_of(sp, last.k, rank);
        int delta = INT32_MIN;
        for (int k = 0; k < 2; ++k)
            for (int r = 0; r < world; ++r) {
                const int b2 = base_of(sp, k, r);
                if ((((bl + 1 - b2) % per) + per) % per == 0) delta = (bl + 1 - b2) / per;
            }
        CDP_REQUIRE(delta != INT32_MIN, "ZeRO-CDP frames: successor use not found");
        const FrameWait f{stage_t0[sp] + 1, stage_t1[sp] + 1, bl, last.dt, delta, per};
        L("zero_frame_wait", 0, 0, s, [&] {
            zero_frame_wait_kernel<<<1, 32, 0, s>>>(f, ring, (const int *)&ctrl_dev.as<Control>()->step);
            CDP_CUDA(cudaGetLastError());
        });
    }
    void zdone(int tensor, int kindFB, cudaStream_t s, int step_delta = 0) {
        if (!zero || sizing) return;
        const ZeroUse z = zuse(tensor, kindFB);
        L("zero_done", 0, 0, s, [&] {
            zero_done_kernel<<<1, 1, 0, s>>>(z, ring, tensor + 1, (const int *)&ctrl_dev.as<Control>()->step,
                                             step_delta);
            CDP_CUDA(cudaGetLastError());
        });
    }

    template <int K>
    void pull_tensor(int tensor, int p, cudaStream_t s) {
        if (zero) {
            zrecv<K>(tensor, 0, s);
            return;
        }
        if (rank == world - 1 || world == 1 || allreduce) return;
        const TensorSpec &ts = tens[tensor];
        const int vslot = vs(tensor, p);
        if (sizing) return;
        CDP_REQUIRE(upd_ring && upd_theta[vslot], "pull outside a connected multi-GPU trainer");
        CTensor w = ts.kind == T_BN ? CTensor{} : wcv[vslot][tensor];
        if (!chain.empty()) {  // forwarding along the reader order (pull chain)
            const int st = ts.stage - 1, pr = chain[size_t(st) * 2], sc = chain[size_t(st) * 2 + 1];
            RingFlags *pf = pr < 0 ? upd_ring : reinterpret_cast<RingFlags *>(peers[pr]);
            const float *src = pr < 0 ? upd_theta[vslot] + ts.base : peer_theta(pr, vslot) + foff[tensor];
            L("pull_wait", 0, 0, s, [&] {
                chain_wait_kernel<<<1, 32, 0, s>>>(pf, pr < 0 ? 1 : 0, ring, tensor + 1, ts.fresh, sc >= 0 ? 1 : 0,
                                                   (const int *)&ctrl_dev.as<Control>()->step);
                CDP_CUDA(cudaGetLastError());
            });
            L("pull", 0, double(ts.n) * (4 + 4 + esz()), s, [&] {
                launch_pdl(chain_pull_kernel<K>, dim3(blocks_for(ts.n, 1024)), dim3(256), 0, s, src,
                           thp(vslot, tensor), ts.n, std::max(ts.cols, 1), w, pf, pr < 0 ? 1 : 0, ring, tensor + 1,
                           ts.fresh, (const int *)&ctrl_dev.as<Control>()->step,
                           cta_counters.as<unsigned>() + kMaxStages, trace ? 1 : 0);
            });
            return;
        }
        L("pull_wait", 0, 0, s, [&] {
            pull_wait_kernel<<<1, 32, 0, s>>>(upd_ring, ring, tensor + 1, ts.fresh,
                                              (const int *)&ctrl_dev.as<Control>()->step);
            CDP_CUDA(cudaGetLastError());
        });
        L("pull", 0, double(ts.n) * (4 + 4 + esz()), s, [&] {
            launch_pdl(pull_tensor_kernel<K>, dim3(blocks_for(ts.n, 1024)), dim3(256), 0, s,
                       (const float *)(upd_theta[vslot] + ts.base), thp(vslot, tensor), ts.n,
                       std::max(ts.cols, 1), w, upd_ring, ring, tensor + 1, ts.fresh,
                       (const int *)&ctrl_dev.as<Control>()->step, cta_counters.as<unsigned>() + kMaxStages,
                       trace ? 1 : 0);
        });
    }

    // Weight hop of conv ci on the hop stream once its dy is ready (and, for a
    // stale read on the updater, once its data gradient has read the old copy).
    template <int K>
    void hop_conv(int ci, int p, cudaEvent_t dy_ready, cudaEvent_t dgrad_done) {
        ConvL &c = convs[ci];
        wait(hs, dy_ready);
        bn_hop(ci, p, hs);
        zdone(c.tb, 1, hs);
        if (dgrad_done && (zero || (!tens[c.tw].fresh && last_updater()))) wait(hs, dgrad_done);
        if (!dgrad_done) zrecv<K>(c.tw, 1, hs);  // the stem: its weight's only backward access is the hop
        conv_wgrad_hop<K>(ci, p, hs);
        zdone(c.tw, 1, hs);
    }

    template <int K>
    void record_step(int p) {
        kernels_per_step = 0;
        flops_per_step = 0.0;
        zero_bytes_per_step = 0;
        zwin_done.assign(size_t(world) * 2, 0);
        cudaEvent_t fork = ev(main);
        wait(cs, fork);
        wait(hs, fork);
        wait(ps, fork);
        // parameter pulls run ahead on their own stream (their waits for the updater block only that
        // stream); each forward waits for its own tensor's pull only.  ZeRO-CDP state copies stay on
        // the compute stream (their use-window order is the protocol).
        forward<K>(p, cs, [&](int tensor) {
            if (zero || rank == world - 1 || world == 1 || allreduce) {
                pull_tensor<K>(tensor, p, cs);
                return;
            }
            pull_tensor<K>(tensor, p, ps);
            wait(cs, ev(ps));
        });
        // loss + classifier backward
        Flags *fl = flags_dev.as<Flags>();
        const int nt = std::max(32, round_up(B, 32));
        const size_t lsm = sizeof(double) * nt + sizeof(float) * B * classes;
        if (classes <= 64 && lsm <= 48 * 1024) {
            L("loss", 0, 0, cs, [&] {
                launch_pdl(loss_kernel<K>, dim3(1), dim3(nt), lsm, cs, (const float *)z.as<float>(), B, classes,
                           loss_kind, (const int *)perm_dev.as<int>(), (const int *)data_lab.as<int>(),
                           (const float *)nullptr, dz.view(), loss_dev.as<double>(), &fl->loss);
            });
        } else {
            L("loss", 0, 0, cs, [&] {
                launch_pdl(xent_rows_kernel<K>, dim3(B), dim3(256), 0, cs, (const float *)z.as<float>(), B, classes,
                           (const int *)perm_dev.as<int>(), (const int *)data_lab.as<int>(), dz.view(),
                           loss_rows.as<double>());
            });
            L("loss_sum", 0, 0, cs, [&] {
                launch_pdl(loss_sum_kernel, dim3(1), dim3(1), 0, cs, (const double *)loss_rows.as<double>(), B,
                           loss_dev.as<double>(), &fl->loss);
            });
        }
        cudaEvent_t dz_ready = ev(cs);
        typename EpiDgradLinear::Params dep{dpooled.as<float>(), fc_in};
        const int vfc = vs(fc_t, p);
        zrecv<K>(fc_t, 1, cs);
        rec(fc_t, A_BWD, 0, vfc, cs);
        gemm<K, false, false, EpiDgradLinear>("fc_dgrad", 32, wcv[vfc][fc_t], dz.view(), fc_in, B, classes, dep,
                                              cs, false);
        rec(fc_t, A_BWD, 1, vfc, cs);
        cudaEvent_t fc_dgrad_done = ev(cs);
        wait(hs, dz_ready);
        if (zero || (!tens[fc_t].fresh && last_updater())) wait(hs, fc_dgrad_done);
        {
            HopParams hp = hop_params(fc_t, p);
            hop_wait(hp, hs);
            traced_update(fc_t, p, hp.mode == 2 || hp.mode == 3, hs, [&] {
                gemm<K, true, true, EpiWgrad<K>>("fc_wgrad_hop", 64, pooled.view(), dz.view(), fc_in + 1, classes, B,
                                                 hp, hs, true);
            });
            zdone(fc_t, 1, hs);
        }
        void *G0 = gbuf[0].p, *G1 = gbuf[1].p, *G2 = gbuf[2].p, *G3 = gbuf[3].p;
        // pool backward -> gradient w.r.t. the last activation (G0 holds the block-output gradient)
        const int la = blocks.empty() ? stem_act : blocks.back().a_out;
        const int HW = int(act_P[la] / B);
        L("avgpool_bwd", 0, double(act_P[la]) * fc_in * ysz(), cs, [&] {
            launch_pdl(avgpool_backward_kernel<K>, dim3(blocks_for(act_P[la] * fc_in / 4)), dim3(256), 0, cs,
                       (const float *)dpooled.as<float>(), fc_in, B, HW, fc_in, G0, acts[la].view());
        });
        for (int bi = int(blocks.size()) - 1; bi >= 0; --bi) {
            BlockL &b = blocks[bi];
            const int n = int(b.convs.size());
            // last BN (+ projection BN): g' = G0, already masked by the block output's ReLU by its producer
            // (the average-pool backward, or the next block's input data gradient)
            bn_backward<K>(b.convs[n - 1], b.ds, p, G0, CTensor{}, cs);
            cudaEvent_t dy_last = ev(cs);
            // projection shortcut first: its data gradient is folded into the first conv's
            if (b.ds >= 0) {
                conv_dgrad<K>(b.ds, vs(convs[b.ds].tw, p), G3, cs);
                cudaEvent_t dg = ev(cs);
                hop_conv<K>(b.ds, p, dy_last, dg);
            }
            void *chain[2] = {G1, G2};
            cudaEvent_t dy_next = dy_last;
            for (int i = n - 1; i >= 0; --i) {
                const int ci = b.convs[i];
                if (i > 0) {
                    void *out = chain[(n - 1 - i) & 1];
                    conv_dgrad<K>(ci, vs(convs[ci].tw, p), out, cs);
                    cudaEvent_t dg = ev(cs);
                    hop_conv<K>(ci, p, dy_next, dg);
                    bn_backward<K>(b.convs[i - 1], -1, p, out, acts[b.mid[i - 1]].view(), cs);
                    dy_next = ev(cs);
                } else {
                    // block input gradient = main branch + shortcut branch, written over G0 and masked by
                    // the previous block's output ReLU (its BN backward and residual then read no mask)
                    conv_dgrad<K>(ci, vs(convs[ci].tw, p), G0, cs, b.ds >= 0 ? G3 : G0, CTensor{},
                                  acts[b.a_in].view());
                    cudaEvent_t dg = ev(cs);
                    hop_conv<K>(ci, p, dy_next, dg);
                }
            }
        }
        // stem (gradient w.r.t. the stem output / max-pool output in G0)
        ConvL &c0 = convs[stem];
        const void *gs = G0;
        if (pool_act >= 0) {
            const int a = stem_act, o = pool_act;
            L("maxpool_bwd", 0, double(act_P[o]) * act_C[o] * (1 + ysz()) + double(act_P[a]) * act_C[a] * ysz(), cs,
              [&] {
                launch_pdl(maxpool_bwd_owner_kernel<K>, dim3(blocks_for(act_P[o] * act_C[o] / 8)), dim3(256), 0, cs,
                           (const void *)G0, (const uint8_t *)pool_arg.as<uint8_t>(), B, act_H[a], act_W[a],
                           act_C[a], act_H[o], act_W[o], G1);
            });
            gs = G1;
        }
        bn_backward<K>(stem, -1, p, gs, acts[stem_act].view(), cs);
        cudaEvent_t dy0 = ev(cs);
        hop_conv<K>(stem, p, dy0, nullptr);
        // join + bookkeeping
        wait(main, ev(cs));
        wait(main, ev(hs));
        wait(main, ev(ps));
        L("finish_step", 0, 0, main, [&] {
            finish_step_kernel_rn<<<1, 1, 0, main>>>(loss_dev.as<double>(), flags_dev.as<Flags>(),
                                                     hist_loss.as<double>(), hist_flags.as<Flags>(), hist_cap,
                                                     &ctrl_dev.as<Control>()->step);
            CDP_CUDA(cudaGetLastError());
        });
        (void)c0;
    }

    // ZeRO-CDP end of a run: a backward of the last step may follow (in the plan's use
    // order) a forward of the NEXT step on another rank; publish those forward uses of
    // step t (= the next, unlaunched step) after their own predecessors, without compute.
    void zero_drain() {
        if (!zero) return;
        // stage the control block of step t (the next, unlaunched step) asynchronously: no host
        // synchronisation here (other ranks' drains may be what this rank's last step waits for)
        std::vector<int> ident(B, 0);
        stage_control(ident.data(), 0.f);
        if (frames) {
            // the next step's forward state copies a frame reuse of this step waits for (zero.py
            // frame_drain_plan: w4's B2 hands its state to w1's F4 of step t + 1 at N = 4), in use order,
            // with their explicit frame waits; the other forwards only publish as with full replicas
            CDP_REQUIRE(!drained, "ZeRO-CDP frames: the run was already drained");
            const int per = 2 * world;
            auto base_of = [&](int st0, int k) { return ztab[((size_t(st0) * 2 + k) * world + rank) * 3]; };
            for (int st = 1; st <= world; ++st) {
                const int *row = nullptr;
                for (size_t k = 0; k + 5 <= zdrain.size(); k += 5)
                    if (zdrain[k] == st) row = &zdrain[k];
                if (row) {
                    if (row[1] >= 0) {
                        const FrameWait f{stage_t0[row[1]] + 1, stage_t1[row[1]] + 1, base_of(row[1], row[2]), row[3],
                                          row[4], per};
                        L("zero_frame_wait", 0, 0, main, [&] {
                            zero_frame_wait_kernel<<<1, 32, 0, main>>>(f, ring,
                                                                       (const int *)&ctrl_dev.as<Control>()->step);
                            CDP_CUDA(cudaGetLastError());
                        });
                    }
                    for (int k = stage_t0[st - 1]; k < stage_t1[st - 1]; ++k) {
                        if (kind == 0)
                            zrecv<0>(k, 0, main, 0, true, false);
                        else
                            zrecv<1>(k, 0, main, 0, true, false);
                        zdone(k, 0, main);
                    }
                    continue;
                }
                for (int k = stage_t0[st - 1]; k < stage_t1[st - 1]; ++k) {
                    bool needed = false;
                    for (int j = 0; j < world; ++j) {
                        const int *e = &ztab[((size_t(st - 1) * 2 + 1) * world + j) * 3];
                        needed |= (e[1] == rank && e[2] == 1);
                    }
                    if (!needed) continue;
                    if (kind == 0)
                        zrecv<0>(k, 0, main, 0, false);
                    else
                        zrecv<1>(k, 0, main, 0, false);
                    zdone(k, 0, main);
                }
            }
            drained = true;
            return;
        }
        for (size_t k = 0; k < tens.size(); ++k) {
            const int tensor = int(k);
            // only forwards some other rank's backward of the last step waits for (zero.py drain_units)
            const int st = tens[k].stage - 1;
            bool needed = false;
            for (int j = 0; j < world; ++j) {
                const int *e = &ztab[((size_t(st) * 2 + 1) * world + j) * 3];
                needed |= (e[1] == rank && e[2] == 1);
            }
            if (!needed) continue;
            if (kind == 0)
                zrecv<0>(tensor, 0, main, 0, false);
            else
                zrecv<1>(tensor, 0, main, 0, false);
            zdone(tensor, 0, main);
        }
    }

    void capture() {
        for (auto &e : exec)
            if (e) {
                CDP_CUDA(cudaGraphExecDestroy(e));
                e = nullptr;
            }
        for (auto e : events) cudaEventDestroy(e);
        events.clear();
        for (int p = 0; p < 2; ++p) {
            cudaGraph_t g;
            CDP_CUDA(cudaStreamBeginCapture(main, cudaStreamCaptureModeThreadLocal));
            try {
                if (kind == 0)
                    record_step<0>(p);
                else
                    record_step<1>(p);
            } catch (...) {
                cudaEvent_t a, b, c;
                cudaEventCreateWithFlags(&a, cudaEventDisableTiming);
                cudaEventCreateWithFlags(&b, cudaEventDisableTiming);
                cudaEventCreateWithFlags(&c, cudaEventDisableTiming);
                cudaEventRecord(a, cs);
                cudaEventRecord(b, hs);
                cudaEventRecord(c, ps);
                cudaStreamWaitEvent(main, a, 0);
                cudaStreamWaitEvent(main, b, 0);
                cudaStreamWaitEvent(main, c, 0);
                if (cudaStreamEndCapture(main, &g) == cudaSuccess && g) cudaGraphDestroy(g);
                cudaEventDestroy(a);
                cudaEventDestroy(b);
                cudaEventDestroy(c);
                cudaGetLastError();
                throw;
            }
            CDP_CUDA(cudaStreamEndCapture(main, &g));
            CDP_CUDA(cudaGraphInstantiate(&exec[p], g, 0));
            CDP_CUDA(cudaGraphDestroy(g));
        }
    }

    // ---------------------------------------------------------------- params / steps
    void pack_slot(int slot) {
        for (size_t i = 0; i < tens.size(); ++i) {
            const TensorSpec &ts = tens[i];
            if (ts.kind == T_BN) continue;
            if (kind == 0)
                pack_tensor_kernel<0><<<blocks_for(ts.n), 256, 0, main>>>(thp(slot, int(i)), ts.n, ts.cols,
                                                                          wcv[slot][i]);
            else
                pack_tensor_kernel<1><<<blocks_for(ts.n), 256, 0, main>>>(thp(slot, int(i)), ts.n, ts.cols,
                                                                          wcv[slot][i]);
            CDP_CUDA(cudaGetLastError());
        }
    }

    // Repack the compute copies of tensors [t0, t1) of theta slot `which` (0 current, 1 previous)
    // after its fp32 values were written from outside (the ZeRO-DP baseline's NCCL broadcast).
    void pack_range(int which, int t0, int t1) {
        CDP_REQUIRE(t0 >= 0 && t0 <= t1 && t1 <= int(tens.size()), "tensor range out of bounds");
        const int slot = which == 0 ? (t & 1) : ((t & 1) ^ 1);
        for (int i = t0; i < t1; ++i) {
            const TensorSpec &ts = tens[i];
            if (ts.kind == T_BN) continue;
            if (kind == 0)
                pack_tensor_kernel<0><<<blocks_for(ts.n), 256, 0, main>>>(thp(slot, int(i)), ts.n, ts.cols,
                                                                          wcv[slot][i]);
            else
                pack_tensor_kernel<1><<<blocks_for(ts.n), 256, 0, main>>>(thp(slot, int(i)), ts.n, ts.cols,
                                                                          wcv[slot][i]);
            CDP_CUDA(cudaGetLastError());
        }
    }

    void set_params(int which, const float *host) {
        if (frames) {  // the initial state every step-1 use without predecessor loads (both version slots)
            CDP_REQUIRE(which < 0 && t == 1, "ZeRO-CDP frames: set_params(-1) before the first step only");
            std::memcpy(init_host, host, size_t(P) * 4);
            std::memset(init_host + P, 0, size_t(P) * 4);
            for (int v = 0; v < 2; ++v) {
                std::vector<uint32_t> tag(kMaxStages, uint32_t(v == 0 ? t : t - 1));
                CDP_CUDA(cudaMemcpy(ring->vtag[v == 0 ? (t & 1) : ((t & 1) ^ 1)], tag.data(), kMaxStages * 4,
                                    cudaMemcpyHostToDevice));
            }
            return;
        }
        for (int v = 0; v < 2; ++v) {
            if (which >= 0 && v != which) continue;
            const int slot = v == 0 ? (t & 1) : ((t & 1) ^ 1);
            CDP_CUDA(cudaMemcpyAsync(theta[slot], host, size_t(P) * 4, cudaMemcpyHostToDevice, main));
            pack_slot(slot);
            // version tags: the current slot holds theta_t, the other theta_{t-1} (ref engine.py:8-10)
            std::vector<uint32_t> tag(kMaxStages, uint32_t(v == 0 ? t : t - 1));
            CDP_CUDA(cudaMemcpy(ring->vtag[slot], tag.data(), kMaxStages * 4, cudaMemcpyHostToDevice));
        }
        CDP_CUDA(cudaStreamSynchronize(main));
    }

    void get_params(int which, float *host) {
        CDP_REQUIRE(!frames, "ZeRO-CDP frames hold single stages: gather with cdp_resnet_zero_state");
        CDP_CUDA(cudaStreamSynchronize(main));
        const int slot = which == 0 ? (t & 1) : ((t & 1) ^ 1);
        CDP_CUDA(cudaMemcpy(host, theta[slot], size_t(P) * 4, cudaMemcpyDeviceToHost));
    }

    // ZeRO-CDP frames: this rank's frame contents in the full parameter layout (every tensor, valid or
    // not) and its last finished use index per tensor (the holder of a stage's newest state is the rank
    // with the largest one).
    void zero_state(int which, float *host, uint32_t *last_use) {
        CDP_REQUIRE(frames, "zero_state: ZeRO-CDP frames only");
        CDP_CUDA(cudaDeviceSynchronize());
        const int slot = which == 0 ? (t & 1) : ((t & 1) ^ 1);
        for (size_t i = 0; i < tens.size(); ++i)
            CDP_CUDA(cudaMemcpy(host + tens[i].base, thp(slot, int(i)), size_t(tens[i].n) * 4, cudaMemcpyDeviceToHost));
        CDP_CUDA(cudaMemcpy(last_use, ring->zdone, tens.size() * 4, cudaMemcpyDeviceToHost));
    }

    void stage_control(const int *perm, float lr) {
        const int k = stage_next;
        stage_next = (stage_next + 1) % RING_N;
        CDP_CUDA(cudaEventSynchronize(stage_ev[k]));
        uint8_t *blk = stage_host + size_t(k) * stage_bytes;
        Control *c = reinterpret_cast<Control *>(blk);
        c->lr = lr;
        c->step = t;
        std::memcpy(blk + sizeof(Control), perm, size_t(B) * 4);
        CDP_CUDA(cudaMemcpyAsync(ctrl_dev.p, blk, sizeof(Control), cudaMemcpyHostToDevice, main));
        CDP_CUDA(cudaMemcpyAsync(perm_dev.p, blk + sizeof(Control), size_t(B) * 4, cudaMemcpyHostToDevice, main));
        CDP_CUDA(cudaEventRecord(stage_ev[k], main));
    }

    void step(const int *perm, float lr) {
        CDP_REQUIRE(!drained, "ZeRO-CDP frames: a drained run cannot continue (its last states sit in next-step "
                              "forward frames); gather the parameters and start a new run");
        stage_control(perm, lr);
        CDP_CUDA(cudaGraphLaunch(exec[t & 1], main));
        ++t;
    }

    // End-to-end step: this step's images / labels come from host memory (copied
    // H2D inside the step, into dataset rows 0..B-1), then the step runs on them.
    void step_host_batch(const float *x, const int32_t *labels, float lr) {
        const size_t img = size_t(Hin) * Win * Cin0;
        CDP_CUDA(cudaMemcpyAsync(data_x.p, x, size_t(B) * img * 4, cudaMemcpyHostToDevice, main));
        CDP_CUDA(cudaMemcpyAsync(data_lab.p, labels, size_t(B) * 4, cudaMemcpyHostToDevice, main));
        std::vector<int> ident(B);
        for (int i = 0; i < B; ++i) ident[i] = i;
        step(ident.data(), lr);
    }

    // Pipelined end-to-end step: the H2D copy of this step's batch runs on a copy stream into dataset
    // rows [slot * B, slot * B + B) (two slots), so it overlaps the previous step's compute; the step
    // waits for its copy, the copy into a slot waits for the step that last read it, and the loss is
    // read back (D2H, into pinned memory) after every step.
    void step_host_batch_async(const float *x, const int32_t *labels, float lr, int slot) {
        CDP_REQUIRE(slot == 0 || slot == 1, "input slot 0 or 1");
        CDP_REQUIRE(n_samples >= 2 * B, "the pipelined input needs 2 micro-batches of dataset rows");
        if (!cps) {
            CDP_CUDA(cudaStreamCreateWithFlags(&cps, cudaStreamNonBlocking));
            for (auto *e : {&in_ev[0], &in_ev[1], &done_ev[0], &done_ev[1]})
                CDP_CUDA(cudaEventCreateWithFlags(e, cudaEventDisableTiming));
            CDP_CUDA(cudaMallocHost(&loss_host, 2 * sizeof(double)));
        }
        const size_t img = size_t(Hin) * Win * Cin0;
        CDP_CUDA(cudaStreamWaitEvent(cps, done_ev[slot], 0));
        CDP_CUDA(cudaMemcpyAsync(data_x.as<float>() + size_t(slot) * B * img, x, size_t(B) * img * 4,
                                 cudaMemcpyHostToDevice, cps));
        CDP_CUDA(cudaMemcpyAsync(data_lab.as<int32_t>() + size_t(slot) * B, labels, size_t(B) * 4,
                                 cudaMemcpyHostToDevice, cps));
        CDP_CUDA(cudaEventRecord(in_ev[slot], cps));
        CDP_CUDA(cudaStreamWaitEvent(main, in_ev[slot], 0));
        std::vector<int> rows(B);
        for (int i = 0; i < B; ++i) rows[i] = slot * B + i;
        step(rows.data(), lr);
        CDP_CUDA(cudaEventRecord(done_ev[slot], main));
        CDP_CUDA(cudaMemcpyAsync(loss_host + slot, loss_dev.p, 8, cudaMemcpyDeviceToHost, main));
    }

    // One real training step run eagerly (not from the graph) with timing events
    // around every launch; returns the per-launch records.
    // serial: every launch on one stream (clean per-kernel durations, no overlap).
    void profile_step(const int *perm, float lr, bool serial) {
        stage_control(perm, lr);
        clear_oprecs();
        instr = true;
        cudaStream_t saved_cs = cs, saved_hs = hs, saved_ps = ps;
        if (serial) cs = hs = ps = main;
        try {
            if (kind == 0)
                record_step<0>(t & 1);
            else
                record_step<1>(t & 1);
        } catch (...) {
            instr = false;
            cs = saved_cs;
            hs = saved_hs;
            ps = saved_ps;
            throw;
        }
        cs = saved_cs;
        hs = saved_hs;
        ps = saved_ps;
        instr = false;
        ++t;
        CDP_CUDA(cudaStreamSynchronize(main));
        CDP_CUDA(cudaDeviceSynchronize());
    }
};

}  // namespace cdp

using namespace cdp;

struct cdp_resnet {
    std::unique_ptr<ResNetTrainer> impl;
};

extern "C" int cdp_resnet_create_rank(int n_layers, const int32_t *widths, const int32_t *depths, int block_kind,
                                      int stem_kind, int in_channels, int height, int width, int classes,
                                      int micro_batch, int world, int rank, const int32_t *tensor_stage,
                                      const uint8_t *stage_fresh, int dtype, float momentum, float weight_decay,
                                      int n_samples, const float *x, const int32_t *labels,
                                      const int32_t *zero_table, int options, cdp_resnet **out) {
    return guarded([&] {
        CDP_REQUIRE(dtype == CDP_DTYPE_FP32 || dtype == CDP_DTYPE_BF16, "bad dtype");
        CDP_REQUIRE(world >= 1 && rank >= 0 && rank < world, "bad rank / world");
        CDP_REQUIRE(micro_batch >= 1 && micro_batch <= 256, "micro-batch must be in [1, 256]");
        CDP_REQUIRE(n_layers >= 1 && n_layers <= 8, "1..8 residual stages");
        CDP_REQUIRE(block_kind == 0 || block_kind == 1, "block_kind: 0 basic, 1 bottleneck");
        CDP_REQUIRE(stem_kind == 0 || stem_kind == 1, "stem_kind: 0 CIFAR 3x3, 1 ImageNet 7x7 + max pool");
        CDP_REQUIRE(in_channels == 3, "stem input channels: 3 (RGB)");
        for (int l = 0; l < n_layers; ++l)
            CDP_REQUIRE(widths[l] % 64 == 0 && widths[l] <= 512, "widths: multiples of 64 up to 512");
        auto tr = std::make_unique<ResNetTrainer>();
        tr->kind = dtype == CDP_DTYPE_BF16 ? 0 : 1;
        tr->B = micro_batch;
        tr->block_kind = block_kind;
        tr->stem_kind = stem_kind;
        tr->Cin0 = in_channels;
        tr->Hin = height;
        tr->Win = width;
        tr->classes = classes;
        tr->momentum = momentum;
        tr->wd = weight_decay;
        tr->rank = rank;
        tr->world = world;
        tr->n_samples = std::max(n_samples, micro_batch);
        tr->allreduce = (options & 1) != 0;
        tr->trace = (options & 2) != 0;
        CDP_REQUIRE(!(tr->allreduce && tr->trace), "trace mode covers the CDP / DP ring step, not the all-reduce baseline");
        if (tr->trace) {
            tr->tlog = DevBuf(size_t(ResNetTrainer::kTraceCap) * kTraceWords * 4);
            tr->tcur = DevBuf(4);
        }
        CDP_REQUIRE(!(tr->allreduce && zero_table), "the DP all-reduce baseline and ZeRO-CDP are exclusive");
        if (zero_table && world > 1) {
            tr->zero = true;
            tr->frames = (options & 4) == 0;  // options bit 2: full replicas (state copied, nothing freed)
            tr->ztab.assign(zero_table, zero_table + size_t(world) * 2 * world * 3);
            for (int k = 0; k < world * 2 * world; ++k) {
                CDP_REQUIRE(tr->ztab[k * 3 + 1] >= 0 && tr->ztab[k * 3 + 1] < world, "ZeRO table: bad source rank");
                CDP_REQUIRE(tr->ztab[k * 3 + 2] >= -1 && tr->ztab[k * 3 + 2] <= 1, "ZeRO table: bad step offset");
            }
        }
        const int HWC = height * width * in_channels;
        tr->data_x = DevBuf(size_t(tr->n_samples) * HWC * 4);
        tr->data_lab = DevBuf(size_t(tr->n_samples) * 4);
        if (x) CDP_CUDA(cudaMemcpy(tr->data_x.p, x, size_t(n_samples) * HWC * 4, cudaMemcpyHostToDevice));
        if (labels) CDP_CUDA(cudaMemcpy(tr->data_lab.p, labels, size_t(n_samples) * 4, cudaMemcpyHostToDevice));
        tr->stage_in = tensor_stage;
        tr->build(widths, depths, n_layers);
        tr->stage_in = nullptr;
        for (size_t i = 0; i < tr->tens.size(); ++i) {
            const int st = tensor_stage[i];
            CDP_REQUIRE(st >= 1 && st <= world, "tensor stage out of range");
            tr->tens[i].stage = st;
            tr->tens[i].fresh = stage_fresh[st - 1] != 0;
        }
        *out = new cdp_resnet{std::move(tr)};
    });
}

extern "C" int cdp_resnet_info(cdp_resnet *tr, int64_t *n_params, int *n_tensors, int64_t *tensor_base,
                               int32_t *tensor_kind) {
    return guarded([&] {
        auto &m = *tr->impl;
        *n_params = m.P;
        *n_tensors = int(m.tens.size());
        if (tensor_base)
            for (size_t i = 0; i < m.tens.size(); ++i) tensor_base[i] = m.tens[i].base;
        if (tensor_kind)
            for (size_t i = 0; i < m.tens.size(); ++i) tensor_kind[i] = m.tens[i].kind;
    });
}

extern "C" int cdp_resnet_region(cdp_resnet *tr, void **base) {
    return guarded([&] { *base = tr->impl->region.p; });
}

extern "C" int cdp_resnet_ipc_handle(cdp_resnet *tr, void *handle64) {
    return guarded([&] {
        cudaIpcMemHandle_t h;
        CDP_CUDA(cudaIpcGetMemHandle(&h, tr->impl->region.p));
        std::memcpy(handle64, &h, sizeof(h));
    });
}

extern "C" int cdp_resnet_connect(cdp_resnet *tr, void *const *regions) {
    return guarded([&] {
        auto &m = *tr->impl;
        auto at = [&](int r) { return static_cast<uint8_t *>(regions[r]); };
        if (m.rank > 0) {
            m.prev_ring = reinterpret_cast<RingFlags *>(at(m.rank - 1));
            m.prev_partial = reinterpret_cast<float *>(at(m.rank - 1) + m.region_off) + 2 * m.th_stride;
        }
        m.peers.assign(size_t(m.world), nullptr);
        for (int r = 0; r < m.world; ++r) m.peers[r] = at(r);
        const int u = m.world - 1;
        m.upd_ring = reinterpret_cast<RingFlags *>(at(u));
        m.upd_theta[0] = reinterpret_cast<float *>(at(u) + m.region_off);
        m.upd_theta[1] = m.upd_theta[0] + m.Pp;
        m.capture();
    });
}

extern "C" void cdp_resnet_destroy(cdp_resnet *tr) {
    if (tr) {
        cudaDeviceSynchronize();
        delete tr;
    }
}

extern "C" int cdp_resnet_set_params(cdp_resnet *tr, int which, const float *theta) {
    return guarded([&] { tr->impl->set_params(which, theta); });
}

extern "C" int cdp_resnet_get_params(cdp_resnet *tr, int which, float *theta) {
    return guarded([&] { tr->impl->get_params(which, theta); });
}

extern "C" int cdp_resnet_step(cdp_resnet *tr, const int32_t *perm, float lr) {
    return guarded([&] { tr->impl->step(perm, lr); });
}

extern "C" int cdp_resnet_step_host_batch(cdp_resnet *tr, const float *x, const int32_t *labels, float lr) {
    return guarded([&] { tr->impl->step_host_batch(x, labels, lr); });
}

extern "C" int cdp_resnet_step_host_batch_async(cdp_resnet *tr, const float *x, const int32_t *labels, float lr,
                                                int slot) {
    return guarded([&] { tr->impl->step_host_batch_async(x, labels, lr, slot); });
}

extern "C" int cdp_resnet_apply_update(cdp_resnet *tr) {
    return guarded([&] { tr->impl->apply_update(); });
}

extern "C" int cdp_resnet_apply_update_range(cdp_resnet *tr, int first_tensor, int end_tensor) {
    return guarded([&] { tr->impl->apply_update(first_tensor, end_tensor); });
}

extern "C" int cdp_resnet_pack_range(cdp_resnet *tr, int which, int first_tensor, int end_tensor) {
    return guarded([&] { tr->impl->pack_range(which, first_tensor, end_tensor); });
}

extern "C" int cdp_resnet_partial(cdp_resnet *tr, void **ptr, size_t *n) {
    return guarded([&] {
        *ptr = tr->impl->partial;
        *n = size_t(tr->impl->P);
    });
}

extern "C" int cdp_resnet_stream(cdp_resnet *tr, void **stream) {
    return guarded([&] { *stream = tr->impl->main; });
}

extern "C" int cdp_resnet_pull_chain(cdp_resnet *tr, const int32_t *pred_succ, int n_stages) {
    return guarded([&] {
        auto &m = *tr->impl;
        CDP_REQUIRE(!m.exec[0], "the pull chain is set before connect (graph capture)");
        CDP_REQUIRE(n_stages == 0 || (n_stages == m.world && pred_succ), "pull chain: one row per stage");
        CDP_REQUIRE(!m.zero && !m.allreduce, "pull chain: CDP ring runs only");
        for (int k = 0; k < 2 * n_stages; ++k)
            CDP_REQUIRE(pred_succ[k] >= -1 && pred_succ[k] < m.world - 1 && pred_succ[k] != m.rank,
                        "pull chain: ranks of other readers");
        m.chain.assign(pred_succ, pred_succ + size_t(n_stages) * 2);
    });
}

extern "C" int cdp_resnet_zero_drain_plan(cdp_resnet *tr, const int32_t *rows, int n_rows) {
    return guarded([&] {
        CDP_REQUIRE(n_rows >= 0 && (n_rows == 0 || rows), "drain plan rows");
        tr->impl->zdrain.assign(rows, rows + size_t(n_rows) * 5);
    });
}

extern "C" int cdp_resnet_zero_state(cdp_resnet *tr, int which, float *theta, uint32_t *last_use) {
    return guarded([&] { tr->impl->zero_state(which, theta, last_use); });
}

extern "C" int cdp_resnet_zero_drain(cdp_resnet *tr) {
    return guarded([&] { tr->impl->zero_drain(); });
}

extern "C" int cdp_resnet_last_loss(cdp_resnet *tr, double *loss) {
    return guarded([&] {
        auto &m = *tr->impl;
        CDP_CUDA(cudaStreamSynchronize(m.main));
        CDP_CUDA(cudaMemcpy(loss, m.loss_dev.p, 8, cudaMemcpyDeviceToHost));
    });
}

extern "C" int cdp_resnet_profile_step(cdp_resnet *tr, const int32_t *perm, float lr, int serial, int max_ops,
                                       char *names, int name_len, double *flops, double *bytes, float *ms,
                                       int *n_ops) {
    return guarded([&] {
        auto &m = *tr->impl;
        m.profile_step(perm, lr, serial != 0);
        const int n = std::min<int>(max_ops, int(m.oprecs.size()));
        *n_ops = int(m.oprecs.size());
        for (int i = 0; i < n; ++i) {
            const OpRec &o = m.oprecs[i];
            std::strncpy(names + size_t(i) * name_len, o.name.c_str(), name_len - 1);
            names[size_t(i) * name_len + name_len - 1] = 0;
            flops[i] = o.flops;
            bytes[i] = o.bytes;
            CDP_CUDA(cudaEventElapsedTime(&ms[i], o.a, o.b));
        }
    });
}

extern "C" int cdp_resnet_history(cdp_resnet *tr, int max, double *losses, uint32_t *flags, int *count) {
    return guarded([&] {
        auto &m = *tr->impl;
        CDP_CUDA(cudaStreamSynchronize(m.main));
        const int c = m.t - 1;
        *count = c;
        const int n = std::min({c, max, m.hist_cap});
        std::vector<double> l(m.hist_cap);
        std::vector<Flags> f(m.hist_cap);
        CDP_CUDA(cudaMemcpy(l.data(), m.hist_loss.p, size_t(m.hist_cap) * 8, cudaMemcpyDeviceToHost));
        CDP_CUDA(cudaMemcpy(f.data(), m.hist_flags.p, size_t(m.hist_cap) * sizeof(Flags), cudaMemcpyDeviceToHost));
        for (int i = 0; i < n; ++i) {
            const int k = (c - n + i) % m.hist_cap;
            losses[i] = l[k];
            flags[3 * i] = f[k].grad;
            flags[3 * i + 1] = f[k].loss;
            flags[3 * i + 2] = f[k].upd;
        }
    });
}

extern "C" int cdp_resnet_sync(cdp_resnet *tr) {
    return guarded([&] { CDP_CUDA(cudaStreamSynchronize(tr->impl->main)); });
}

extern "C" int cdp_resnet_ring_error(cdp_resnet *tr, int *err) {
    return guarded([&] {
        CDP_CUDA(cudaStreamSynchronize(tr->impl->main));
        uint32_t e = 0;
        CDP_CUDA(cudaMemcpy(&e, &tr->impl->ring->err, 4, cudaMemcpyDeviceToHost));
        *err = int(e);
    });
}

extern "C" int cdp_resnet_stats(cdp_resnet *tr, int64_t *out, int n_out) {
    // [0] activation bytes (activations, conv outputs, dy, stem record), [1] parameter-state bytes,
    // [2] kernels / step, [3] tensor-core flops / step, [4] gradient scratch bytes,
    // [5] ZeRO-CDP state bytes received per step
    return guarded([&] {
        auto &m = *tr->impl;
        int64_t act = int64_t(m.cols.hi.bytes + m.cols.lo.bytes);
        for (auto &a : m.acts) act += int64_t(a.hi.bytes + a.lo.bytes);
        for (auto &c : m.convs) act += int64_t(c.y.bytes + c.dy.hi.bytes + c.dy.lo.bytes);
        // persistent parameter state: theta slots, momentum, compute copies (frames in ZeRO-CDP mode) and
        // the gradient partial sum
        int64_t par = int64_t(m.th_stride) * (m.vel ? 12 : 8) + int64_t(m.Pp) * 4;
        for (int v = 0; v < 2; ++v) {
            for (auto &w : m.wc[v]) par += int64_t(w.hi.bytes + w.lo.bytes);
            par += int64_t(m.wcpool[v][0].bytes + m.wcpool[v][1].bytes);
        }
        int64_t scratch = 0;
        for (auto &g : m.gbuf) scratch += int64_t(g.bytes);
        int64_t vals[6] = {act, par, m.kernels_per_step, int64_t(m.flops_per_step), scratch, m.zero_bytes_per_step};
        for (int i = 0; i < n_out && i < 6; ++i) out[i] = vals[i];
    });
}

// Device address / size / row pitch of one internal buffer (tests and diagnostics read them
// after cdp_resnet_sync; names in include/cdp_b200.h).
extern "C" int cdp_resnet_buffer(cdp_resnet *tr, const char *name, int index, void **ptr, size_t *bytes, int *ld) {
    return guarded([&] {
        auto &m = *tr->impl;
        const std::string n(name);
        const DevBuf *d = nullptr;
        int l = 0;
        auto conv = [&]() -> ConvL & {
            CDP_REQUIRE(index >= 0 && index < int(m.convs.size()), "conv index out of range");
            return m.convs[index];
        };
        auto cb = [&](const CBuf &c, bool lo) {
            d = lo ? &c.lo : &c.hi;
            l = c.ld;
        };
        if (n == "wc_hi" || n == "wc_lo") {
            CDP_REQUIRE(index >= 0 && index < 2 * int(m.tens.size()), "wc index: slot * n_tensors + tensor");
            cb(m.wc[index / int(m.tens.size())][index % int(m.tens.size())], n == "wc_lo");
        } else if (n == "act_hi" || n == "act_lo") {
            CDP_REQUIRE(index >= 0 && index < int(m.acts.size()), "activation index out of range");
            cb(m.acts[index], n == "act_lo");
        } else if (n == "dy_hi" || n == "dy_lo") {
            cb(conv().dy, n == "dy_lo");
        } else if (n == "y") {
            d = &conv().y;
        } else if (n == "mean") {
            d = &conv().mean;
        } else if (n == "rstd") {
            d = &conv().rstd;
        } else if (n == "dgamma") {
            d = &conv().dgamma;
        } else if (n == "dbeta") {
            d = &conv().dbeta;
        } else if (n == "gbuf") {
            CDP_REQUIRE(index >= 0 && index < 4, "gbuf index 0..3");
            d = &m.gbuf[index];
        } else if (n == "dpooled") {
            d = &m.dpooled;
        } else if (n == "z") {
            d = &m.z;
        } else if (n == "pooled_hi" || n == "pooled_lo") {
            cb(m.pooled, n == "pooled_lo");
        } else if (n == "dz_hi" || n == "dz_lo") {
            cb(m.dz, n == "dz_lo");
        } else if (n == "theta") {  // index 0: current slot, 1: previous (fp32, P values)
            CDP_REQUIRE(index == 0 || index == 1, "theta index: 0 current, 1 previous");
            const int slot = index == 0 ? (m.t & 1) : ((m.t & 1) ^ 1);
            *ptr = m.theta[slot];
            *bytes = size_t(m.P) * 4;
            *ld = 0;
            return;
        } else if (n == "region") {
            d = &m.region;
        } else if (n == "pool_arg") {
            d = &m.pool_arg;
        } else {
            throw CdpError("unknown buffer name " + n);
        }
        *ptr = d->p;
        *bytes = d->bytes;
        *ld = l;
    });
}

extern "C" int cdp_resnet_trace(cdp_resnet *tr, uint32_t *records, int max_records, int *count) {
    return guarded([&] {
        auto &m = *tr->impl;
        CDP_REQUIRE(m.trace, "trainer created without the trace option");
        CDP_CUDA(cudaStreamSynchronize(m.main));
        uint32_t n = 0;
        CDP_CUDA(cudaMemcpy(&n, m.tcur.p, 4, cudaMemcpyDeviceToHost));
        CDP_REQUIRE(n <= ResNetTrainer::kTraceCap, "trace buffer overflow: read the records more often");
        *count = int(n);
        const int k = std::min<int>(int(n), max_records);
        if (k > 0) CDP_CUDA(cudaMemcpy(records, m.tlog.p, size_t(k) * kTraceWords * 4, cudaMemcpyDeviceToHost));
        CDP_CUDA(cudaMemset(m.tcur.p, 0, 4));
    });
}

extern "C" int cdp_resnet_mark(cdp_resnet *tr, int k) {
    return guarded([&] {
        auto &m = *tr->impl;
        while (int(m.marks.size()) <= k) {
            cudaEvent_t e;
            CDP_CUDA(cudaEventCreate(&e));
            m.marks.push_back(e);
        }
        CDP_CUDA(cudaEventRecord(m.marks[k], m.main));
    });
}

extern "C" int cdp_resnet_elapsed(cdp_resnet *tr, int a, int b, float *ms) {
    return guarded([&] {
        auto &m = *tr->impl;
        CDP_CUDA(cudaEventSynchronize(m.marks[b]));
        CDP_CUDA(cudaEventElapsedTime(ms, m.marks[a], m.marks[b]));
    });
}

extern "C" int cdp_resnet_flush_l2(cdp_resnet *tr) {
    return guarded([&] {
        auto &m = *tr->impl;
        if (!m.flush_buf.p) m.flush_buf = DevBuf(size_t(256) << 20);
        CDP_CUDA(cudaMemsetAsync(m.flush_buf.p, m.t & 0xff, m.flush_buf.bytes, m.main));
    });
}
