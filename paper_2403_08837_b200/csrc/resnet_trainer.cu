// Device-resident CDP training step for BasicBlock ResNets (BASELINE configs[1]:
// ResNet-18, CIFAR-10 shape 32x32, one micro-batch per GPU).
//
// Same step semantics as the MLP trainer (ref training/engine.py:66-116 with
// the per-stage version rule, gradient hops w_i -> w_{i+1}, fused update on
// the last worker, parameter pulls) with convolutional layer compute:
//   conv  = im2col + tcgen05 GEMM (rows = output pixels, NHWC), fp32 output;
//   BN    = training-mode batch statistics (fp64 fixed-order reductions),
//           affine + residual + ReLU fused into one pass;
//   dgrad = tcgen05 GEMM into im2col space + deterministic col2im gather;
//   wgrad = tcgen05 GEMM (split-K over pixels) whose epilogue is the hop /
//           SGD update of the weight tensor (EpiWgrad, as for the MLP);
//   BN gamma|beta hop / update by a vector kernel.
// One worker per process (rank mode; world = 1 is plain single-GPU training).
// Hop units are parameter tensors in torchvision order: conv weights
// [R*S*Cin][Cout], BN [gamma(C) | beta(C)], classifier [[W^T]; b] = [C+1][classes].
#include <cuda_bf16.h>

#include <array>
#include <cstring>
#include <functional>
#include <memory>
#include <string>
#include <vector>

#include "../../include/cdp_b200.h"
#include "conv_kernels.cuh"
#include "gemm_launch.cuh"
#include "trainer_common.cuh"

namespace cdp {

namespace {

enum TensorKind { T_CONV = 0, T_BN = 1, T_FC = 2 };

struct TensorSpec {
    int kind;
    int64_t base, n;
    int rows, cols;  // GEMM view for conv / fc
    int stage;       // 1-based stage (version unit)
    int fresh;       // this worker reads the current version of this tensor's stage
};

struct ConvL {
    int cin, cout, R, S, stride, pad, H, W, Ho, Wo, K;
    int tw, tb;  // tensor indices of the conv weight and its BN
    int64_t P;   // output rows B*Ho*Wo
    DevBuf y, mean, rstd, dbeta, dgamma;
    CBuf dy;     // gradient w.r.t. the conv output (GEMM operand)
};

struct BlockL {
    int c1, c2, ds;         // conv indices (ds = -1: identity shortcut)
    int a_in, a1, a_out;    // activation indices
};

template <int KIND>
__global__ void gather_image_kernel_k(const float *__restrict__ data, int HWC, int C, const int *perm, CTensor out) {
    ptx::griddep_wait();
    ptx::griddep_launch();
    const int s = blockIdx.x;
    const float *src = data + size_t(perm[s]) * HWC;
    const int HW = HWC / C;
    for (int i = threadIdx.x; i < HWC; i += blockDim.x) {
        const int pix = i / C, c = i % C;
        Fmt<KIND>::store(out.hi, out.lo, (size_t(s) * HW + pix) * out.ld + c, src[i]);
    }
}

// Copy one parameter tensor of version v from the updater (peer HBM) into the
// local slot, packing the GEMM compute copy when it has one; count the pull.
template <int KIND>
__global__ void pull_tensor_kernel(const float *__restrict__ src, float *dst, int64_t n, int cols, CTensor wc,
                                   RingFlags *updater, RingFlags *own, int unit, int fresh, const int *step,
                                   unsigned *cta_counter) {
    ptx::griddep_wait();
    ptx::griddep_launch();
    const int t = *step;
    const uint32_t v = uint32_t(fresh ? t : t - 1);
    if (v <= 1) return;
    if (threadIdx.x == 0) spin_ge(&updater->updated[unit - 1], v, &own->err);
    __syncthreads();
    for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < n; i += int64_t(gridDim.x) * blockDim.x) {
        const float x = __ldcv(src + i);
        dst[i] = x;
        if (wc.hi) Fmt<KIND>::store(wc.hi, wc.lo, size_t(i / cols) * wc.ld + i % cols, x);
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        __threadfence_system();
        if (atomicAdd(&cta_counter[unit - 1], 1u) == gridDim.x - 1) {
            cta_counter[unit - 1] = 0;
            atomicAdd_system(&updater->pulled[unit - 1][v & 1], 1u);
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

}  // namespace

struct ResNetTrainer {
    // ---------------------------------------------------------------- config
    int kind = 0, B = 0, Hin = 32, Win = 32, Cin0 = 3, classes = 10, loss_kind = 1;
    float momentum = 0.f, wd = 0.f, eps = 1e-5f;
    int rank = 0, world = 1;
    std::vector<TensorSpec> tens;
    std::vector<ConvL> convs;
    std::vector<BlockL> blocks;
    int stem = 0, fc_t = -1, fc_in = 0;
    int64_t P = 0, Pp = 0;

    // ---------------------------------------------------------------- state
    DevBuf region, vel, cta_counters;
    float *theta[2] = {nullptr, nullptr};
    float *partial = nullptr;
    RingFlags *ring = nullptr;
    size_t region_off = 0;
    RingFlags *prev_ring = nullptr, *upd_ring = nullptr;
    float *prev_partial = nullptr, *upd_theta[2] = {nullptr, nullptr};
    std::vector<CBuf> wc[2];   // per tensor (empty CBuf for BN)
    std::vector<CBuf> acts;    // activations (compute format)
    std::vector<DevBuf> gacts; // fp32 gradients w.r.t. activations
    std::vector<int> act_C;
    std::vector<int64_t> act_P;
    CBuf x_in, cols_c, cols_h, pooled, dz;
    DevBuf dcols, dpooled, z, gtmp, bn_partial, loss_dev;
    DevBuf ws_c, cnt_c, ws_h, cnt_h;
    size_t ws_c_floats = 0, ws_h_floats = 0;
    DevBuf data_x, data_lab, ctrl_dev, perm_dev, flags_dev, hist_loss, hist_flags;
    int n_samples = 0;
    static constexpr int RING_N = 16;
    uint8_t *stage_host = nullptr;
    size_t stage_bytes = 0;
    cudaEvent_t stage_ev[RING_N] = {};
    int stage_next = 0;
    int hist_cap = 1 << 14;
    cudaStream_t main = nullptr, cs = nullptr, hs = nullptr;
    std::vector<cudaEvent_t> events;
    cudaGraphExec_t exec[2] = {nullptr, nullptr};
    int t = 1;
    int kernels_per_step = 0;
    std::vector<cudaEvent_t> marks;
    DevBuf flush_buf;

    ~ResNetTrainer() {
        for (auto &e : exec)
            if (e) cudaGraphExecDestroy(e);
        for (auto e : events) cudaEventDestroy(e);
        for (auto e : marks) cudaEventDestroy(e);
        for (auto e : stage_ev)
            if (e) cudaEventDestroy(e);
        if (stage_host) cudaFreeHost(stage_host);
        for (auto s : {main, cs, hs})
            if (s) cudaStreamDestroy(s);
    }

    // ---------------------------------------------------------------- model
    int add_tensor(int k, int64_t n, int rows, int cols) {
        int64_t base = tens.empty() ? 0 : tens.back().base + tens.back().n;
        tens.push_back(TensorSpec{k, base, n, rows, cols, 1, 1});
        return int(tens.size()) - 1;
    }

    int add_act(int64_t rows, int C) {
        acts.push_back(make_cbuf(kind, int(rows), C));
        gacts.emplace_back(size_t(rows) * C * 4);
        act_C.push_back(C);
        act_P.push_back(rows);
        return int(acts.size()) - 1;
    }

    int add_conv(int cin, int cout, int R, int stride, int H, int W) {
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
        c.tw = add_tensor(T_CONV, int64_t(c.K) * cout, c.K, cout);
        c.tb = add_tensor(T_BN, 2 * int64_t(cout), 0, 0);
        convs.push_back(std::move(c));
        return int(convs.size()) - 1;
    }

    void build(const int *widths, const int *depths, int n_layers) {
        int H = Hin, W = Win;
        x_in = make_cbuf(kind, B * H * W, Cin0);
        stem = add_conv(Cin0, widths[0], 3, 1, H, W);
        int a = add_act(int64_t(B) * H * W, widths[0]);
        int cin = widths[0];
        for (int l = 0; l < n_layers; ++l) {
            for (int d = 0; d < depths[l]; ++d) {
                const int stride = (l > 0 && d == 0) ? 2 : 1;
                const int cout = widths[l];
                BlockL b{};
                b.a_in = a;
                b.c1 = add_conv(cin, cout, 3, stride, H, W);
                const int Ho = convs[b.c1].Ho, Wo = convs[b.c1].Wo;
                b.a1 = add_act(int64_t(B) * Ho * Wo, cout);
                b.c2 = add_conv(cout, cout, 3, 1, Ho, Wo);
                b.ds = (stride != 1 || cin != cout) ? add_conv(cin, cout, 1, stride, H, W) : -1;
                b.a_out = add_act(int64_t(B) * Ho * Wo, cout);
                blocks.push_back(b);
                a = b.a_out;
                cin = cout;
                H = Ho;
                W = Wo;
            }
        }
        fc_in = cin;
        fc_t = add_tensor(T_FC, int64_t(cin + 1) * classes, cin + 1, classes);
        P = tens.back().base + tens.back().n;
        // ---- buffers
        int64_t max_cols = 0, max_dc = 0;
        for (auto &c : convs) {
            c.y = DevBuf(size_t(c.P) * c.cout * 4);
            c.mean = DevBuf(c.cout * 4);
            c.rstd = DevBuf(c.cout * 4);
            c.dbeta = DevBuf(c.cout * 4);
            c.dgamma = DevBuf(c.cout * 4);
            c.dy = make_cbuf(kind, int(c.P), c.cout);
            max_cols = std::max<int64_t>(max_cols, c.P * round_up(c.K, 16));
            max_dc = std::max<int64_t>(max_dc, c.P * round_up(c.K, 16));
        }
        int64_t maxP = 0;
        for (auto &c : convs) maxP = std::max(maxP, c.P);
        cols_c = make_cbuf(kind, 1, int(max_cols));  // viewed with per-conv ld
        cols_h = make_cbuf(kind, 1, int(max_cols));
        dcols = DevBuf(size_t(max_dc) * 4);
        gtmp = DevBuf(size_t(maxP) * 512 * 4 + size_t(maxP) * 64 * 4);
        bn_partial = DevBuf(size_t((maxP + kBnRowsPerBlock - 1) / kBnRowsPerBlock) * 512 * 2 * 8);
        pooled = make_cbuf(kind, B, fc_in + 1);
        dz = make_cbuf(kind, B, classes);
        dpooled = DevBuf(size_t(B) * fc_in * 4);
        z = DevBuf(size_t(B) * classes * 4);
        loss_dev = DevBuf(8);
        // shared region: RingFlags | theta0 | theta1 | partial
        region_off = (sizeof(RingFlags) + 255) / 256 * 256;
        Pp = (P + 63) / 64 * 64;
        region = DevBuf(region_off + size_t(Pp) * 4 * 3);
        ring = region.as<RingFlags>();
        theta[0] = reinterpret_cast<float *>(region.as<uint8_t>() + region_off);
        theta[1] = theta[0] + Pp;
        partial = theta[1] + Pp;
        if (momentum != 0.f) vel = DevBuf(size_t(P) * 4);
        cta_counters = DevBuf(2 * kMaxStages * 4);
        for (int v = 0; v < 2; ++v)
            for (auto &ts : tens) wc[v].push_back(ts.kind == T_BN ? CBuf{} : make_cbuf(kind, ts.rows, ts.cols));
        CDP_REQUIRE(int(tens.size()) <= kMaxStages, "too many parameter tensors for the ring flags");
        // split-K workspaces (sized by a dry run of the split heuristic)
        for (auto &c : convs) {
            ws_c_floats = std::max(ws_c_floats, ws_need(c.P, c.cout, bn_cout(c.cout), c.K));
            ws_c_floats = std::max(ws_c_floats, ws_need(c.P, c.K, 128, c.cout));
            ws_h_floats = std::max(ws_h_floats, ws_need(c.K, c.cout, 64, c.P));
        }
        ws_h_floats = std::max(ws_h_floats, ws_need(fc_in + 1, classes, 64, B));
        ws_c = DevBuf(std::max<size_t>(ws_c_floats, 1) * 4);
        ws_h = DevBuf(std::max<size_t>(ws_h_floats, 1) * 4);
        cnt_c = DevBuf(1 << 16);
        cnt_h = DevBuf(1 << 16);
        CDP_CUDA(cudaStreamCreateWithFlags(&main, cudaStreamNonBlocking));
        CDP_CUDA(cudaStreamCreateWithFlags(&cs, cudaStreamNonBlocking));
        CDP_CUDA(cudaStreamCreateWithFlags(&hs, cudaStreamNonBlocking));
        ctrl_dev = DevBuf(sizeof(Control));
        perm_dev = DevBuf(size_t(B) * 4);
        flags_dev = DevBuf(sizeof(Flags));
        hist_loss = DevBuf(size_t(hist_cap) * 8);
        hist_flags = DevBuf(size_t(hist_cap) * sizeof(Flags));
        stage_bytes = (sizeof(Control) + size_t(B) * 4 + 255) / 256 * 256;
        CDP_CUDA(cudaMallocHost(&stage_host, stage_bytes * RING_N));
        for (auto &e : stage_ev) CDP_CUDA(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
    }

    // ---------------------------------------------------------------- GEMM plumbing
    static int bn_cout(int cout) { return std::min(256, cout); }
    int splits_for(int64_t M, int64_t N, int BN, int64_t K) const {
        const int bk = kind == 0 ? 64 : 32, nseg = kind == 0 ? 1 : 3;
        const int64_t total = ((K + bk - 1) / bk) * nseg;
        const int64_t tiles = ((M + 127) / 128) * ((N + BN - 1) / BN);
        int64_t s = std::max<int64_t>(1, (2 * 148 + tiles - 1) / tiles);
        s = std::min(s, total);
        const int64_t per = (total + s - 1) / s;
        return int((total + per - 1) / per);
    }
    size_t ws_need(int64_t M, int64_t N, int BN, int64_t K) const {
        const int s = splits_for(M, N, BN, K);
        return s <= 1 ? 0 : size_t((M + 127) / 128) * ((N + BN - 1) / BN) * s * 128 * BN;
    }

    template <int K>
    static int segs(const Operand &a_hi, const Operand &a_lo, const Operand &b_hi, const Operand &b_lo, Operand *A,
                    Operand *Bo) {
        if (K == 0) {
            A[0] = a_hi, Bo[0] = b_hi;
            return 1;
        }
        A[0] = a_hi, Bo[0] = b_hi;
        A[1] = a_hi, Bo[1] = b_lo;
        A[2] = a_lo, Bo[2] = b_hi;
        return 3;
    }
    static Operand opnd(const CTensor &t, bool lo, bool mn, int64_t mn_ext, int64_t k_ext) {
        return Operand{lo ? t.lo : t.hi, mn, uint64_t(mn_ext), uint64_t(k_ext), uint64_t(t.ld)};
    }

    template <int K, bool AMN, bool BMN, class Epi>
    void gemm(int BN, const CTensor &a, int64_t am, int64_t ak, const CTensor &b, int64_t bn_, int64_t bk, int64_t M,
              int64_t N, int64_t Kd, const typename Epi::Params &ep, cudaStream_t s, bool hop_stream) {
        Operand A[3], Bo[3];
        const int nseg = segs<K>(opnd(a, false, AMN, am, ak), opnd(a, true, AMN, am, ak), opnd(b, false, BMN, bn_, bk),
                                 opnd(b, true, BMN, bn_, bk), A, Bo);
        const int splits = splits_for(M, N, BN, Kd);
        float *ws = hop_stream ? ws_h.as<float>() : ws_c.as<float>();
        int *cnt = hop_stream ? cnt_h.as<int>() : cnt_c.as<int>();
        const size_t cap = hop_stream ? ws_h_floats : ws_c_floats;
#define CDP_RG(BN_)                                                                                             \
    case BN_:                                                                                                   \
        if constexpr ((!BMN || BN_ % (K == 0 ? 64 : 32) == 0) && (!Epi::kTile || BN_ <= 64)) {                  \
            GemmPlan p = plan_gemm<K, BN_, AMN, BMN>(A, Bo, nseg, int(M), int(N), int(Kd), splits, ws, cnt);     \
            CDP_REQUIRE(gemm_ws_floats(p, BN_) <= cap, "split-K workspace too small");                        \
            launch_gemm<K, BN_, AMN, BMN, Epi>(p, ep, s);                                                      \
            ++kernels_per_step;                                                                                \
            return;                                                                                            \
        }                                                                                                       \
        break;
        switch (BN) {
            CDP_RG(32)
            CDP_RG(64)
            CDP_RG(128)
            CDP_RG(256)
            default:
                break;
        }
#undef CDP_RG
        throw CdpError("unsupported GEMM tile width " + std::to_string(BN));
    }

    CTensor cols_view(const CBuf &c, int K) const { return CTensor{c.hi.p, c.lo.p, round_up(K, 16)}; }
    static int blocks_for(int64_t n, int per = 256) { return int(std::min<int64_t>(4 * 148, (n + per - 1) / per)); }

    // ---------------------------------------------------------------- forward pieces
    template <int K>
    void conv_forward(int ci, const CTensor &in, int vslot, cudaStream_t s) {
        ConvL &c = convs[ci];
        const CTensor cv = cols_view(cols_c, c.K);
        launch_pdl(im2col_kernel<K>, dim3(blocks_for(c.P, 1)), dim3(128), 0, s, in, B, c.H, c.W, c.cin, c.R, c.S,
                   c.stride, c.pad, c.Ho, c.Wo, cv);
        ++kernels_per_step;
        EpiRowF32::Params ep{c.y.as<float>(), c.cout};
        gemm<K, false, true, EpiRowF32>(bn_cout(c.cout), cv, c.P, c.K, wc[vslot][c.tw].view(), c.cout, c.K, c.P,
                                         c.cout, c.K, ep, s, false);
        bn_stats(c, s);
    }

    void bn_stats(ConvL &c, cudaStream_t s) {
        const int nblk = int((c.P + kBnRowsPerBlock - 1) / kBnRowsPerBlock);
        launch_pdl(bn_partial_kernel<0>, dim3(nblk), dim3(std::min(256, c.cout)), 0, s, (const float *)c.y.as<float>(),
                   c.cout, c.P, c.cout, 0, (const float *)nullptr, 0, CTensor{}, (const float *)nullptr,
                   (const float *)nullptr, bn_partial.as<double>());
        launch_pdl(bn_finalize_kernel, dim3((c.cout + 127) / 128), dim3(128), 0, s,
                   (const double *)bn_partial.as<double>(), nblk, c.cout, c.P, 0, eps, c.mean.as<float>(),
                   c.rstd.as<float>());
        kernels_per_step += 2;
    }

    const float *gamma(int ci, int vslot) const { return theta[vslot] + tens[convs[ci].tb].base; }
    const float *beta(int ci, int vslot) const { return theta[vslot] + tens[convs[ci].tb].base + convs[ci].cout; }
    int vs(int tensor, int p) const { return tens[tensor].fresh ? p : (p ^ 1); }

    template <int K>
    void forward(int p, cudaStream_t s, const std::function<void(int)> &pull) {
        // input
        launch_pdl(gather_image_kernel_k<K>, dim3(B), dim3(256), 0, s, (const float *)data_x.as<float>(),
                   Hin * Win * Cin0, Cin0, (const int *)perm_dev.as<int>(), x_in.view());
        ++kernels_per_step;
        // stem
        ConvL &c0 = convs[stem];
        pull(c0.tw);
        pull(c0.tb);
        conv_forward<K>(stem, x_in.view(), vs(c0.tw, p), s);
        bn_apply<K>(stem, vs(c0.tb, p), BnResidual{}, 1, acts[0].view(), s);
        for (auto &b : blocks) {
            ConvL &c1 = convs[b.c1];
            pull(c1.tw);
            pull(c1.tb);
            conv_forward<K>(b.c1, acts[b.a_in].view(), vs(c1.tw, p), s);
            bn_apply<K>(b.c1, vs(c1.tb, p), BnResidual{}, 1, acts[b.a1].view(), s);
            ConvL &c2 = convs[b.c2];
            pull(c2.tw);
            pull(c2.tb);
            conv_forward<K>(b.c2, acts[b.a1].view(), vs(c2.tw, p), s);
            BnResidual res{};
            if (b.ds >= 0) {
                ConvL &cd = convs[b.ds];
                pull(cd.tw);
                pull(cd.tb);
                conv_forward<K>(b.ds, acts[b.a_in].view(), vs(cd.tw, p), s);
                res.x = cd.y.as<float>();
                res.ldx = cd.cout;
                res.mean = cd.mean.as<float>();
                res.rstd = cd.rstd.as<float>();
                res.gamma = gamma(b.ds, vs(cd.tb, p));
                res.beta = beta(b.ds, vs(cd.tb, p));
            } else {
                res.act = acts[b.a_in].view();
            }
            bn_apply<K>(b.c2, vs(c2.tb, p), res, 1, acts[b.a_out].view(), s);
        }
        // pool + classifier
        const int last = blocks.empty() ? 0 : blocks.back().a_out;
        const int HW = int(act_P[last] / B);
        launch_pdl(avgpool_kernel<K>, dim3(B), dim3(256), 0, s, acts[last].view(), B, HW, fc_in, pooled.view());
        ++kernels_per_step;
        pull(fc_t);
        typename EpiFwd<K>::Params ep{};
        ep.last = 1;
        ep.z = z.as<float>();
        gemm<K, true, false, EpiFwd<K>>(32, wc[vs(fc_t, p)][fc_t].view(), classes, fc_in + 1, pooled.view(), B,
                                         fc_in + 1, classes, B, fc_in + 1, ep, s, false);
    }

    template <int K>
    void bn_apply(int ci, int vslot, const BnResidual &res, int relu, const CTensor &out, cudaStream_t s) {
        ConvL &c = convs[ci];
        launch_pdl(bn_apply_kernel<K>, dim3(blocks_for(c.P * c.cout)), dim3(256), 0, s, (const float *)c.y.as<float>(),
                   c.cout, c.P, c.cout, (const float *)c.mean.as<float>(), (const float *)c.rstd.as<float>(),
                   gamma(ci, vslot), beta(ci, vslot), res, relu, out);
        ++kernels_per_step;
    }

    // ---------------------------------------------------------------- backward pieces
    // BN backward for conv ci: g (fp32, w.r.t. the BN+ReLU output), mask = that output.
    template <int K>
    void bn_backward(int ci, int vslot, const float *g, const CTensor &mask, cudaStream_t s) {
        ConvL &c = convs[ci];
        const int nblk = int((c.P + kBnRowsPerBlock - 1) / kBnRowsPerBlock);
        launch_pdl(bn_partial_kernel<K>, dim3(nblk), dim3(std::min(256, c.cout)), 0, s,
                   (const float *)c.y.as<float>(), c.cout, c.P, c.cout, 1, g, c.cout, mask,
                   (const float *)c.mean.as<float>(), (const float *)c.rstd.as<float>(), bn_partial.as<double>());
        launch_pdl(bn_finalize_kernel, dim3((c.cout + 127) / 128), dim3(128), 0, s,
                   (const double *)bn_partial.as<double>(), nblk, c.cout, c.P, 1, eps, c.dbeta.as<float>(),
                   c.dgamma.as<float>());
        launch_pdl(bn_backward_kernel<K>, dim3(blocks_for(c.P * c.cout)), dim3(256), 0, s,
                   (const float *)c.y.as<float>(), c.cout, c.P, c.cout, (const float *)c.mean.as<float>(),
                   (const float *)c.rstd.as<float>(), gamma(ci, vslot), (const float *)c.dbeta.as<float>(),
                   (const float *)c.dgamma.as<float>(), g, c.cout, mask, c.dy.view());
        kernels_per_step += 3;
    }

    // conv data gradient: dcols = dy . W^T, then col2im into g_in (fp32 [P_in][cin]).
    template <int K>
    void conv_dgrad(int ci, int vslot, float *g_in, cudaStream_t s) {
        ConvL &c = convs[ci];
        const int Kp = round_up(c.K, 16);
        EpiRowF32::Params ep{dcols.as<float>(), Kp};
        gemm<K, false, false, EpiRowF32>(128, c.dy.view(), c.P, c.cout, wc[vslot][c.tw].view(), c.K, c.cout, c.P, c.K,
                                          c.cout, ep, s, false);
        const int64_t nin = int64_t(B) * c.H * c.W * c.cin;
        launch_pdl(col2im_kernel, dim3(blocks_for(nin)), dim3(256), 0, s, (const float *)dcols.as<float>(), Kp, B, c.H,
                   c.W, c.cin, c.R, c.S, c.stride, c.pad, c.Ho, c.Wo, g_in, c.cin);
        ++kernels_per_step;
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
        hp.theta_cur = theta[p];
        hp.theta_new = theta[p ^ 1];
        hp.vel = vel.as<float>();
        hp.lr = &ctrl_dev.as<Control>()->lr;
        hp.momentum = momentum;
        hp.wd = wd;
        hp.n_mb = float(world);
        hp.wc_new = ts.kind == T_BN ? CTensor{} : wc[p ^ 1][tensor].view();
        Flags *fl = flags_dev.as<Flags>();
        hp.grad_flags = &fl->grad;
        hp.upd_flags = &fl->upd;
        hp.sync.enabled = 1;
        hp.sync.n_readers = world - 1;
        hp.sync.step = &ctrl_dev.as<Control>()->step;
        hp.sync.own = ring;
        hp.sync.prev = prev_ring;
        hp.sync.cta_counter = cta_counters.as<unsigned>();
        return hp;
    }

    // weight gradient of conv ci fused with its hop / update (hop stream).
    template <int K>
    void conv_wgrad_hop(int ci, const CTensor &in, int p, cudaStream_t s) {
        ConvL &c = convs[ci];
        const CTensor cv = cols_view(cols_h, c.K);
        launch_pdl(im2col_kernel<K>, dim3(blocks_for(c.P, 1)), dim3(128), 0, s, in, B, c.H, c.W, c.cin, c.R, c.S,
                   c.stride, c.pad, c.Ho, c.Wo, cv);
        ++kernels_per_step;
        HopParams hp = hop_params(c.tw, p);
        gemm<K, true, true, EpiWgrad<K>>(64, cv, c.K, c.P, c.dy.view(), c.cout, c.P, c.K, c.cout, c.P, hp, s, true);
    }

    void bn_hop(int ci, int p, cudaStream_t s) {
        ConvL &c = convs[ci];
        HopParams hp = hop_params(c.tb, p);
        launch_pdl(vector_hop_kernel, dim3(1), dim3(128), 0, s, hp, (const float *)c.dgamma.as<float>(),
                   (const float *)c.dbeta.as<float>(), c.cout);
        ++kernels_per_step;
    }

    // ---------------------------------------------------------------- step capture
    cudaEvent_t ev(cudaStream_t s) {
        cudaEvent_t e;
        CDP_CUDA(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
        events.push_back(e);
        CDP_CUDA(cudaEventRecord(e, s));
        return e;
    }
    void wait(cudaStream_t s, cudaEvent_t e) { CDP_CUDA(cudaStreamWaitEvent(s, e, 0)); }
    bool last_updater() const { return rank == world - 1; }

    template <int K>
    void pull_tensor(int tensor, int p, cudaStream_t s) {
        if (rank == world - 1 || world == 1) return;
        const TensorSpec &ts = tens[tensor];
        const int vslot = vs(tensor, p);
        CDP_REQUIRE(upd_ring && upd_theta[vslot], "pull outside a connected multi-GPU trainer");
        CTensor w = ts.kind == T_BN ? CTensor{} : wc[vslot][tensor].view();
        launch_pdl(pull_tensor_kernel<K>, dim3(blocks_for(ts.n, 1024)), dim3(256), 0, s,
                   (const float *)(upd_theta[vslot] + ts.base), theta[vslot] + ts.base, ts.n, std::max(ts.cols, 1), w,
                   upd_ring, ring, tensor + 1, ts.fresh, (const int *)&ctrl_dev.as<Control>()->step,
                   cta_counters.as<unsigned>() + kMaxStages);
        ++kernels_per_step;
    }

    template <int K>
    void record_step(int p) {
        kernels_per_step = 0;
        cudaEvent_t fork = ev(main);
        wait(cs, fork);
        wait(hs, fork);
        forward<K>(p, cs, [&](int tensor) { pull_tensor<K>(tensor, p, cs); });
        // loss + classifier backward
        Flags *fl = flags_dev.as<Flags>();
        const int nt = std::max(32, round_up(B, 32));
        const size_t lsm = sizeof(double) * nt + sizeof(float) * B * classes;
        launch_pdl(loss_kernel<K>, dim3(1), dim3(nt), lsm, cs, (const float *)z.as<float>(), B, classes, loss_kind,
                   (const int *)perm_dev.as<int>(), (const int *)data_lab.as<int>(), (const float *)nullptr, dz.view(),
                   loss_dev.as<double>(), &fl->loss);
        ++kernels_per_step;
        cudaEvent_t dz_ready = ev(cs);
        typename EpiDgradLinear::Params dep{dpooled.as<float>(), fc_in};
        const int vfc = vs(fc_t, p);
        gemm<K, false, false, EpiDgradLinear>(32, wc[vfc][fc_t].view(), fc_in, classes, dz.view(), B, classes, fc_in,
                                               B, classes, dep, cs, false);
        cudaEvent_t fc_dgrad_done = ev(cs);
        // classifier hop
        wait(hs, dz_ready);
        if (!tens[fc_t].fresh && last_updater()) wait(hs, fc_dgrad_done);
        {
            HopParams hp = hop_params(fc_t, p);
            gemm<K, true, true, EpiWgrad<K>>(64, pooled.view(), fc_in + 1, B, dz.view(), classes, B, fc_in + 1,
                                              classes, B, hp, hs, true);
        }
        // pool backward -> gradient w.r.t. the last activation
        const int last = blocks.back().a_out;
        const int HW = int(act_P[last] / B);
        launch_pdl(avgpool_backward_kernel, dim3(blocks_for(act_P[last] * fc_in)), dim3(256), 0, cs,
                   (const float *)dpooled.as<float>(), fc_in, B, HW, fc_in, gacts[last].as<float>(), fc_in);
        ++kernels_per_step;
        // blocks in reverse
        for (int bi = int(blocks.size()) - 1; bi >= 0; --bi) {
            BlockL &b = blocks[bi];
            ConvL &c1 = convs[b.c1], &c2 = convs[b.c2];
            const float *g_out = gacts[b.a_out].as<float>();
            const CTensor m_out = acts[b.a_out].view();
            // second BN (+ shortcut BN)
            bn_backward<K>(b.c2, vs(c2.tb, p), g_out, m_out, cs);
            cudaEvent_t dy2 = ev(cs);
            cudaEvent_t dyd = nullptr;
            if (b.ds >= 0) {
                bn_backward<K>(b.ds, vs(convs[b.ds].tb, p), g_out, m_out, cs);
                dyd = ev(cs);
            }
            // conv2: data gradient into a1's gradient
            conv_dgrad<K>(b.c2, vs(c2.tw, p), gacts[b.a1].as<float>(), cs);
            cudaEvent_t c2_dg = ev(cs);
            // hops of conv2 / bn2 (and the shortcut) overlap the rest of the block
            wait(hs, dy2);
            bn_hop(b.c2, p, hs);
            if (!tens[c2.tw].fresh && last_updater()) wait(hs, c2_dg);
            conv_wgrad_hop<K>(b.c2, acts[b.a1].view(), p, hs);
            // first BN
            bn_backward<K>(b.c1, vs(c1.tb, p), gacts[b.a1].as<float>(), acts[b.a1].view(), cs);
            cudaEvent_t dy1 = ev(cs);
            // conv1 data gradient -> input gradient (main path) in gtmp
            float *g_in = gacts[b.a_in].as<float>();
            float *g_main = gtmp.as<float>();
            conv_dgrad<K>(b.c1, vs(c1.tw, p), g_main, cs);
            cudaEvent_t c1_dg = ev(cs);
            if (b.ds >= 0) {
                ConvL &cd = convs[b.ds];
                float *g_ds = gtmp.as<float>() + size_t(act_P[b.a_in]) * act_C[b.a_in];
                conv_dgrad<K>(b.ds, vs(cd.tw, p), g_ds, cs);
                cudaEvent_t cd_dg = ev(cs);
                launch_pdl(add_kernel<K>, dim3(blocks_for(act_P[b.a_in] * act_C[b.a_in])), dim3(256), 0, cs,
                           (const float *)g_main, (const float *)g_ds, act_C[b.a_in], act_P[b.a_in], act_C[b.a_in],
                           CTensor{}, g_in);
                ++kernels_per_step;
                wait(hs, dyd);
                bn_hop(b.ds, p, hs);
                if (!tens[cd.tw].fresh && last_updater()) wait(hs, cd_dg);
                conv_wgrad_hop<K>(b.ds, acts[b.a_in].view(), p, hs);
            } else {
                // identity shortcut: g_in = g_main + g_out masked by the block output
                launch_pdl(add_kernel<K>, dim3(blocks_for(act_P[b.a_in] * act_C[b.a_in])), dim3(256), 0, cs,
                           (const float *)g_main, g_out, act_C[b.a_in], act_P[b.a_in], act_C[b.a_in], m_out, g_in);
                ++kernels_per_step;
            }
            cudaEvent_t gin_done = ev(cs);
            (void)gin_done;
            wait(hs, dy1);
            bn_hop(b.c1, p, hs);
            if (!tens[c1.tw].fresh && last_updater()) wait(hs, c1_dg);
            conv_wgrad_hop<K>(b.c1, acts[b.a_in].view(), p, hs);
            // the next (earlier) block's compute reuses gtmp: its dgrad must not race the add above
        }
        // stem
        ConvL &c0 = convs[stem];
        bn_backward<K>(stem, vs(c0.tb, p), gacts[0].as<float>(), acts[0].view(), cs);
        cudaEvent_t dy0 = ev(cs);
        wait(hs, dy0);
        bn_hop(stem, p, hs);
        conv_wgrad_hop<K>(stem, x_in.view(), p, hs);
        // join + bookkeeping
        wait(main, ev(cs));
        wait(main, ev(hs));
        finish_step_kernel_rn<<<1, 1, 0, main>>>(loss_dev.as<double>(), flags_dev.as<Flags>(), hist_loss.as<double>(),
                                                 hist_flags.as<Flags>(), hist_cap, &ctrl_dev.as<Control>()->step);
        CDP_CUDA(cudaGetLastError());
        ++kernels_per_step;
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
                cudaEvent_t a, b;
                cudaEventCreateWithFlags(&a, cudaEventDisableTiming);
                cudaEventCreateWithFlags(&b, cudaEventDisableTiming);
                cudaEventRecord(a, cs);
                cudaEventRecord(b, hs);
                cudaStreamWaitEvent(main, a, 0);
                cudaStreamWaitEvent(main, b, 0);
                if (cudaStreamEndCapture(main, &g) == cudaSuccess && g) cudaGraphDestroy(g);
                cudaEventDestroy(a);
                cudaEventDestroy(b);
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
                pack_tensor_kernel<0><<<blocks_for(ts.n), 256, 0, main>>>(theta[slot] + ts.base, ts.n, ts.cols,
                                                                          wc[slot][i].view());
            else
                pack_tensor_kernel<1><<<blocks_for(ts.n), 256, 0, main>>>(theta[slot] + ts.base, ts.n, ts.cols,
                                                                          wc[slot][i].view());
            CDP_CUDA(cudaGetLastError());
        }
    }

    void set_params(int which, const float *host) {
        for (int v = 0; v < 2; ++v) {
            if (which >= 0 && v != which) continue;
            const int slot = v == 0 ? (t & 1) : ((t & 1) ^ 1);
            CDP_CUDA(cudaMemcpyAsync(theta[slot], host, size_t(P) * 4, cudaMemcpyHostToDevice, main));
            pack_slot(slot);
        }
        CDP_CUDA(cudaStreamSynchronize(main));
    }

    void get_params(int which, float *host) {
        CDP_CUDA(cudaStreamSynchronize(main));
        const int slot = which == 0 ? (t & 1) : ((t & 1) ^ 1);
        CDP_CUDA(cudaMemcpy(host, theta[slot], size_t(P) * 4, cudaMemcpyDeviceToHost));
    }

    void step(const int *perm, float lr) {
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
        CDP_CUDA(cudaGraphLaunch(exec[t & 1], main));
        ++t;
    }
};

}  // namespace cdp

using namespace cdp;

struct cdp_resnet {
    std::unique_ptr<ResNetTrainer> impl;
};

extern "C" int cdp_resnet_create_rank(int n_layers, const int32_t *widths, const int32_t *depths, int in_channels,
                                      int height, int width, int classes, int micro_batch, int world, int rank,
                                      const int32_t *tensor_stage, const uint8_t *stage_fresh, int dtype,
                                      float momentum, float weight_decay, int n_samples, const float *x,
                                      const int32_t *labels, cdp_resnet **out) {
    return guarded([&] {
        CDP_REQUIRE(dtype == CDP_DTYPE_FP32 || dtype == CDP_DTYPE_BF16, "bad dtype");
        CDP_REQUIRE(world >= 1 && rank >= 0 && rank < world, "bad rank / world");
        CDP_REQUIRE(micro_batch >= 1 && micro_batch <= 256, "micro-batch must be in [1, 256]");
        CDP_REQUIRE(n_layers >= 1 && n_layers <= 8, "1..8 residual stages");
        for (int l = 0; l < n_layers; ++l) CDP_REQUIRE(widths[l] % 64 == 0 && widths[l] <= 512, "widths: multiples of 64 up to 512");
        auto tr = std::make_unique<ResNetTrainer>();
        tr->kind = dtype == CDP_DTYPE_BF16 ? 0 : 1;
        tr->B = micro_batch;
        tr->Cin0 = in_channels;
        tr->Hin = height;
        tr->Win = width;
        tr->classes = classes;
        tr->momentum = momentum;
        tr->wd = weight_decay;
        tr->rank = rank;
        tr->world = world;
        tr->build(widths, depths, n_layers);
        for (size_t i = 0; i < tr->tens.size(); ++i) {
            const int st = tensor_stage[i];
            CDP_REQUIRE(st >= 1 && st <= world, "tensor stage out of range");
            tr->tens[i].stage = st;
            tr->tens[i].fresh = stage_fresh[st - 1] != 0;
        }
        tr->n_samples = std::max(n_samples, micro_batch);
        const int HWC = height * width * in_channels;
        tr->data_x = DevBuf(size_t(tr->n_samples) * HWC * 4);
        tr->data_lab = DevBuf(size_t(tr->n_samples) * 4);
        if (x) CDP_CUDA(cudaMemcpy(tr->data_x.p, x, size_t(n_samples) * HWC * 4, cudaMemcpyHostToDevice));
        if (labels) CDP_CUDA(cudaMemcpy(tr->data_lab.p, labels, size_t(n_samples) * 4, cudaMemcpyHostToDevice));
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
            m.prev_partial = reinterpret_cast<float *>(at(m.rank - 1) + m.region_off) + 2 * m.Pp;
        }
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
    // [0] activation bytes (activations, conv outputs, dy), [1] parameter-state bytes, [2] kernels / step
    return guarded([&] {
        auto &m = *tr->impl;
        int64_t act = 0;
        for (auto &a : m.acts) act += int64_t(a.hi.bytes + a.lo.bytes);
        for (auto &c : m.convs) act += int64_t(c.y.bytes + c.dy.hi.bytes + c.dy.lo.bytes);
        int64_t par = int64_t(m.Pp) * 12 + int64_t(m.vel.bytes);
        for (int v = 0; v < 2; ++v)
            for (auto &w : m.wc[v]) par += int64_t(w.hi.bytes + w.lo.bytes);
        int64_t vals[3] = {act, par, m.kernels_per_step};
        for (int i = 0; i < n_out && i < 3; ++i) out[i] = vals[i];
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
