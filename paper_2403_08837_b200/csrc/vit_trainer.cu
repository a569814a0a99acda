// Device-resident CDP training step for Vision Transformers (BASELINE configs[3]:
// ViT-B/16, 224x224), bf16 operands (fp32 mode: tf32 hi + lo pairs, 3xTF32), fp32
// residual stream / master state.
//
// Same step semantics as the other trainers (ref training/engine.py:66-116: the
// per-stage version rule, gradient hops w_i -> w_{i+1} fused into the weight-gradient
// GEMM epilogues, the SGD-momentum update on the last worker, parameter pulls), one
// worker (micro-batch) per process, or N workers on one GPU (cyclic executor).  Layer compute:
//   linear layers  = persistent tcgen05 GEMMs (gemm_pk_kernel, GM_PLAIN) with the bias
//                    folded in by a ones column ([x, 1] . [W; b] = the reference's
//                    flat [W][b] layout); GELU and the residual add fused in epilogues;
//   attention      = fused kernels (attn_kernels.cuh: scores / probabilities in TMEM and
//                    shared memory, bf16), or (fp32 mode, T > 256, CDP_VIT_UNFUSED=1)
//                    batched tcgen05 GEMMs (GM_BATCH) over 4-D TMA views of the fused
//                    qkv buffer {64 dims, tokens, heads, samples} + row softmax kernels;
//   LayerNorm      = warp-per-row kernels, parameter gradients by fixed-order row blocks.
// Hop units (parameter tensors, torchvision order): patch [[W^T]; b], cls, pos, per
// block ln1 [g | b], qkv, proj, ln2, fc1, fc2 (linear [[W^T]; b]), final ln, head.
#include <cuda_bf16.h>

#include <cmath>
#include <cstring>
#include <memory>
#include <string>
#include <vector>

#include "../../include/cdp_b200.h"
#include "attn_kernels.cuh"
#include "gemm_launch.cuh"
#include "rank_common.cuh"
#include "trainer_common.cuh"
#include "vit_kernels.cuh"

namespace cdp {

namespace {

enum VitUnitKind { V_LIN = 0, V_LN = 1, V_VEC = 2 };

inline size_t cbytes(const CBuf &b) { return b.hi.bytes + b.lo.bytes; }  // compute format: hi (+ lo, fp32 mode)

struct VUnit {
    int kind;
    int64_t base, n;
    int rows, cols;  // GEMM view of a linear unit ([in + 1][out])
    int stage, fresh;
};

// Forward record of one transformer block for one micro-batch: its input and everything its
// backward reads.  Lives from the forward that writes its input to the block's backward; slots
// come from the step plan's interval colouring (executor.compile_segment_plan).
struct VRec {
    DevBuf h, hmid;                   // fp32 residual stream: block input, after attention
    DevBuf m1, r1, m2, r2;            // LayerNorm row statistics
    CBuf u1, u2, attn, g1, qkvb, z1;  // LN outputs, attention output, GELU output, qkv, gelu'(FC1 pre-activation)
    CBuf P;                           // unfused attention: softmax probabilities [B*H][T][ldp] (compute format)
    DevBuf lse;                       // fused attention: row log-sum-exp fp32 [B*H][T]
    size_t bytes() const {
        return h.bytes + hmid.bytes + m1.bytes + r1.bytes + m2.bytes + r2.bytes + cbytes(u1) + cbytes(u2) +
               cbytes(attn) + cbytes(g1) + cbytes(qkvb) + z1.hi.bytes + cbytes(P) + lse.bytes;
    }
};
struct ERec {  // embedding record: the patch matrix [x, 1] (the patch weight gradient's operand)
    CBuf patches;
    size_t bytes() const { return cbytes(patches); }
};
struct FRec {  // final record: last block output, final LN statistics / output, logits, dlogits
    DevBuf hL, mf, rf, z;
    CBuf uf, dz;
    size_t bytes() const { return hL.bytes + mf.bytes + rf.bytes + z.bytes + cbytes(uf) + cbytes(dz); }
};
// Backward operands of one block read by the hop stream (weight gradients), plus its LN parameter gradients.
struct VGrad {
    CBuf dz1, dhmc, dqkv;
    DevBuf dg1, db1, dg2, db2;
};
struct VBlock {
    int ln1, qkv, proj, ln2, fc1, fc2;  // unit indices
};
// Gradient carried through one worker's backward: dL/dh (fp32) and its bf16 operand copy.
struct VCarry {
    DevBuf dh;
    CBuf dhc[2];
};
struct VOp {
    int kind, worker, stage;  // 0 = F, 1 = B; 1-based worker / stage
};

struct BView {  // a 4-D TMA view {inner, rows, heads, samples} of a token-major compute-format buffer
    const void *ptr;
    int inner, rows;
    int64_t ld, hs, bs;  // elements
    const void *lo;      // fp32 mode: the lo half (same layout), else null
};
struct COpnd {  // a GEMM operand in compute format: hi (bf16, or tf32-exact fp32) and the fp32 mode's lo half
    Operand hi;
    const void *lo;
};

__global__ void live_probe_kernel(int64_t *ctr, int64_t delta) {  // [0] live record bytes, [1] high-water mark
    ctr[0] += delta;
    if (ctr[0] > ctr[1]) ctr[1] = ctr[0];
}

__global__ void loss_mean_kernel(const double *loss_w, int W, double *loss_out) {  // mean_i loss_i, ascending i
    double a = 0.0;
    for (int i = 0; i < W; ++i) a += loss_w[i];
    *loss_out = a / W;
}

}  // namespace

// KIND 0: bf16 operands (the bench path); KIND 1: fp32 mode (operands as hi + lo tf32 pairs, 3xTF32 tcgen05
// products, unfused attention with fp32 softmax) for fp32-tolerance parity with the restatement.
template <int KIND>
struct VitTrainer {
    static constexpr int ES = KIND == 0 ? 2 : 4;  // compute-format bytes per element
    // ---------------------------------------------------------------- config
    int B = 0, img = 224, P = 16, G = 14, NP = 196, T = 197, D = 768, H = 12, HD = 64, F = 3072, L = 12;
    int classes = 1000, loss_kind = 1;
    float momentum = 0.f, wd = 0.f, eps = 1e-6f;
    int rank = 0, world = 1;  // multi-GPU ring: this process is worker rank + 1 of `world`
    int W = 1;                // workers (micro-batches) run by this process: > 1 = single-GPU cyclic CDP
    std::vector<VUnit> units;
    std::vector<VBlock> blocks;
    int u_patch = 0, u_cls = 0, u_pos = 0, u_ln = 0, u_head = 0;
    int64_t Pn = 0, Pp = 0;
    int R = 0, lds = 0, ldp = 0;
    bool fused_attn = true;
    // step plan (W > 1): ops in timeline order, record slot of (worker, segment), pool sizes
    std::vector<VOp> plan;
    std::vector<std::vector<uint8_t>> freshw;  // [worker][unit]
    std::vector<std::vector<int>> slot;        // [worker][segment 0..L+1]
    int pool[3] = {1, 1, 1};                   // embed, block, final record slots
    std::vector<int> seg_stage;                // [segment] (W > 1)
    bool probe = false;

    // ---------------------------------------------------------------- state
    DevBuf region, cta_counters;
    float *vel = nullptr, *theta[2] = {nullptr, nullptr}, *partial = nullptr;
    RingFlags *ring = nullptr;
    size_t region_off = 0;
    RingFlags *prev_ring = nullptr, *upd_ring = nullptr;
    std::vector<uint8_t *> peer_regions;  // every rank's shared region (the pull chain's sources)
    std::vector<int> chain;               // pull chain per stage (predecessor or -1 = updater, successor or -1)
    float *prev_partial = nullptr, *upd_theta[2] = {nullptr, nullptr};
    std::vector<CBuf> wc[2];
    std::vector<VRec> brec;
    std::vector<ERec> erec;
    std::vector<FRec> frec;
    std::vector<VGrad> grads;   // per block (W == 1: the hop stream lags the compute stream) or one (W > 1)
    std::vector<VCarry> carry;  // per worker
    DevBuf E, loss_w, loss_dev, loss_rows, S, dP, du, duf, dhm, gpos, gcls, lnpart, dgf, dbf, live;
    CBuf dattn, dS, dE;
    DevBuf ws_c, ws_h, cnt_c, cnt_h;
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
    double flops_per_step = 0.0;
    std::vector<cudaEvent_t> marks;
    DevBuf flush_buf;
    bool sizing = false, instr = false;
    bool trace = false;  // version tags + per-access records (tests; rank_common.cuh)
    DevBuf tlog, tcur;
    static constexpr uint32_t kTraceCap = 1u << 16;
    struct OpRec {
        std::string name;
        double flops, bytes;
        cudaEvent_t a, b;
    };
    std::vector<OpRec> oprecs;
    int sms_ = 0;
    int cw = 0;  // worker (0-based) whose segment is being recorded

    ~VitTrainer() {
        for (auto &e : exec)
            if (e) cudaGraphExecDestroy(e);
        for (auto e : events) cudaEventDestroy(e);
        for (auto e : marks) cudaEventDestroy(e);
        clear_oprecs();
        for (auto e : stage_ev)
            if (e) cudaEventDestroy(e);
        if (stage_host) cudaFreeHost(stage_host);
        for (auto s : {main, cs, hs})
            if (s) cudaStreamDestroy(s);
    }
    void clear_oprecs() {
        for (auto &o : oprecs) {
            cudaEventDestroy(o.a);
            cudaEventDestroy(o.b);
        }
        oprecs.clear();
    }
    template <class Fn>
    void L_(const char *name, double flops, double bytes, cudaStream_t s, Fn &&f) {
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
    int sms() {
        if (!sms_) sms_ = num_sms();
        return sms_;
    }
    static int blocks_for(int64_t n, int per = 256) { return int(std::min<int64_t>(8 * 148, (n + per - 1) / per)); }
    // a supported BN covering n (fp32 mode: at most 128, the fp32 operand stages are twice as large)
    static int tile_n(int n) { return n <= 64 ? 64 : (n <= 128 || KIND == 1) ? 128 : 256; }

    // ---------------------------------------------------------------- model
    int add_unit(int kind, int64_t n, int rows, int cols) {
        const int64_t base = units.empty() ? 0 : units.back().base + units.back().n;
        units.push_back(VUnit{kind, base, n, rows, cols, 1, 1});
        return int(units.size()) - 1;
    }
    // segment of a unit: 0 = embedding (patch, cls, pos), 1..L = blocks, L + 1 = final LN + head
    int seg_of_unit(int u) const {
        if (u <= u_pos) return 0;
        if (u >= u_ln) return L + 1;
        return 1 + (u - u_pos - 1) / 6;
    }

    void make_units() {
        G = img / P;
        NP = G * G;
        T = NP + 1;
        HD = D / H;
        CDP_REQUIRE(HD == 64, "head dim must be 64 (one 128-byte TMA chunk)");
        CDP_REQUIRE(D % 64 == 0 && F % 64 == 0 && img % P == 0, "dims: multiples of 64; image a multiple of the patch");
        R = B * T;
        lds = round_up(T, 4);
        ldp = round_up(T, 16);
        // fused attention (attn_kernels.cuh): one key tile, T <= 256 (CDP_VIT_UNFUSED=1: batched GEMMs +
        // row-softmax kernels)
        fused_attn = KIND == 0 && T <= 256 && std::getenv("CDP_VIT_UNFUSED") == nullptr;  // bf16 kernels
        const int K0 = P * P * 3;
        u_patch = add_unit(V_LIN, int64_t(K0 + 1) * D, K0 + 1, D);
        u_cls = add_unit(V_VEC, D, 0, 0);
        u_pos = add_unit(V_VEC, int64_t(T) * D, 0, 0);
        blocks.resize(L);
        for (auto &bl : blocks) {
            bl.ln1 = add_unit(V_LN, 2 * D, 0, 0);
            bl.qkv = add_unit(V_LIN, int64_t(D + 1) * 3 * D, D + 1, 3 * D);
            bl.proj = add_unit(V_LIN, int64_t(D + 1) * D, D + 1, D);
            bl.ln2 = add_unit(V_LN, 2 * D, 0, 0);
            bl.fc1 = add_unit(V_LIN, int64_t(D + 1) * F, D + 1, F);
            bl.fc2 = add_unit(V_LIN, int64_t(F + 1) * D, F + 1, D);
        }
        u_ln = add_unit(V_LN, 2 * D, 0, 0);
        u_head = add_unit(V_LIN, int64_t(D + 1) * classes, D + 1, classes);
        Pn = units.back().base + units.back().n;
        CDP_REQUIRE(int(units.size()) <= kMaxStages, "too many parameter tensors for the ring flags");
    }

    void build() {
        // ---- records (pool sizes from the plan), per-block backward operands, per-worker carries
        auto ones = [&](CBuf &b, int rows, int col) {  // constant 1 in column `col` (bias folding; lo stays 0)
            if (KIND == 0) {
                std::vector<__nv_bfloat16> one(size_t(rows), __float2bfloat16(1.f));
                CDP_CUDA(cudaMemcpy2D(static_cast<__nv_bfloat16 *>(b.hi.p) + col, size_t(b.ld) * 2, one.data(), 2, 2,
                                      size_t(rows), cudaMemcpyHostToDevice));
            } else {
                std::vector<float> one(size_t(rows), 1.f);
                CDP_CUDA(cudaMemcpy2D(static_cast<float *>(b.hi.p) + col, size_t(b.ld) * 4, one.data(), 4, 4,
                                      size_t(rows), cudaMemcpyHostToDevice));
            }
        };
        const int K0 = P * P * 3;
        erec.resize(pool[0]);
        for (auto &e : erec) e.patches = make_cbuf(KIND, B * NP, K0 + 1);
        brec.resize(pool[1]);
        for (auto &y : brec) {
            y.h = DevBuf(size_t(R) * D * 4);
            y.hmid = DevBuf(size_t(R) * D * 4);
            y.m1 = DevBuf(size_t(R) * 4);
            y.r1 = DevBuf(size_t(R) * 4);
            y.m2 = DevBuf(size_t(R) * 4);
            y.r2 = DevBuf(size_t(R) * 4);
            y.u1 = make_cbuf(KIND, R, D + 1);
            y.u2 = make_cbuf(KIND, R, D + 1);
            y.attn = make_cbuf(KIND, R, D + 1);
            ones(y.attn, R, D);
            y.g1 = make_cbuf(KIND, R, F + 1);
            ones(y.g1, R, F);
            y.qkvb = make_cbuf(KIND, R, 3 * D);
            y.z1 = make_cbuf(KIND, R, F);
            if (fused_attn)
                y.lse = DevBuf(size_t(B) * H * T * 4);
            else
                y.P = make_cbuf(KIND, B * H * T, T);  // ld = ldp
        }
        frec.resize(pool[2]);
        for (auto &f : frec) {
            f.hL = DevBuf(size_t(R) * D * 4);
            f.mf = DevBuf(size_t(B) * 4);
            f.rf = DevBuf(size_t(B) * 4);
            f.uf = make_cbuf(KIND, B, D + 1);
            f.z = DevBuf(size_t(B) * classes * 4);
            f.dz = make_cbuf(KIND, B, classes);
        }
        grads.resize(W > 1 ? 1 : L);
        for (auto &g : grads) {
            g.dz1 = make_cbuf(KIND, R, F);
            g.dhmc = make_cbuf(KIND, R, D);
            g.dqkv = make_cbuf(KIND, R, 3 * D);
            for (DevBuf *v : {&g.dg1, &g.db1, &g.dg2, &g.db2}) *v = DevBuf(size_t(D) * 4);
        }
        // W == 1: one dhc per block output (the hop stream reads it after the compute stream moved on);
        // W > 1: two per worker (block parity), the hop stream is joined at every segment
        carry.resize(W);
        for (auto &c : carry) c.dh = DevBuf(size_t(R) * D * 4);
        dhc_layer.resize(W == 1 ? L : 0);
        for (auto &d : dhc_layer) d = make_cbuf(KIND, R, D);
        if (W > 1)
            for (auto &c : carry)
                for (auto &d : c.dhc) d = make_cbuf(KIND, R, D);
        E = DevBuf(size_t(B) * NP * D * 4);
        loss_w = DevBuf(size_t(W) * 8);
        loss_dev = DevBuf(8);
        loss_rows = DevBuf(size_t(B) * 8);
        if (!fused_attn) {
            S = DevBuf(size_t(B) * H * T * lds * 4);
            dP = DevBuf(size_t(B) * H * T * lds * 4);
            dS = make_cbuf(KIND, B * H * T, T);  // ld = ldp
        }
        du = DevBuf(size_t(R) * D * 4);
        duf = DevBuf(size_t(B) * D * 4);
        dhm = DevBuf(size_t(R) * D * 4);
        dattn = make_cbuf(KIND, R, D);
        gpos = DevBuf(size_t(T) * D * 4);
        gcls = DevBuf(size_t(D) * 4);
        dE = make_cbuf(KIND, B * NP, D);
        lnpart = DevBuf(size_t(D) * ((R + kLnBwdRows - 1) / kLnBwdRows) * 16);
        dgf = DevBuf(size_t(D) * 4);
        dbf = DevBuf(size_t(D) * 4);
        live = DevBuf(16);
        // ---- shared region: RingFlags | theta0 | theta1 | partial | momentum
        region_off = (sizeof(RingFlags) + 255) / 256 * 256;
        Pp = (Pn + 63) / 64 * 64;
        region = DevBuf(region_off + size_t(Pp) * 4 * (momentum != 0.f ? 4 : 3));
        ring = region.as<RingFlags>();
        theta[0] = reinterpret_cast<float *>(region.as<uint8_t>() + region_off);
        theta[1] = theta[0] + Pp;
        partial = theta[1] + Pp;
        if (momentum != 0.f) vel = partial + Pp;
        cta_counters = DevBuf(2 * kMaxStages * 4);
        for (int v = 0; v < 2; ++v)
            for (auto &u : units) wc[v].push_back(u.kind == V_LIN ? make_cbuf(KIND, u.rows, u.cols) : CBuf{});
        CDP_CUDA(cudaStreamCreateWithFlags(&main, cudaStreamNonBlocking));
        CDP_CUDA(cudaStreamCreateWithFlags(&cs, cudaStreamNonBlocking));
        CDP_CUDA(cudaStreamCreateWithFlags(&hs, cudaStreamNonBlocking));
        ctrl_dev = DevBuf(sizeof(Control));
        perm_dev = DevBuf(size_t(W) * B * 4);
        flags_dev = DevBuf(sizeof(Flags));
        hist_loss = DevBuf(size_t(hist_cap) * 8);
        hist_flags = DevBuf(size_t(hist_cap) * sizeof(Flags));
        stage_bytes = (sizeof(Control) + size_t(W) * B * 4 + 255) / 256 * 256;
        CDP_CUDA(cudaMallocHost(&stage_host, stage_bytes * RING_N));
        for (auto &e : stage_ev) CDP_CUDA(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
        cnt_c = DevBuf(1 << 18);
        cnt_h = DevBuf(1 << 18);
        sizing = true;
        record_step(0);
        sizing = false;
        for (auto e : events) cudaEventDestroy(e);
        events.clear();
        ws_c = DevBuf(std::max<size_t>(ws_c_floats, 1) * 4);
        ws_h = DevBuf(std::max<size_t>(ws_h_floats, 1) * 4);
    }
    std::vector<CBuf> dhc_layer;
    // bf16 copy of dL/d(output of block l) for the current worker
    const CBuf &dhc(int l) const { return W == 1 ? dhc_layer[l] : carry[cw].dhc[l & 1]; }
    VGrad &grad_of(int l) { return grads[W > 1 ? 0 : l]; }
    int64_t record_bytes(int pool_kind) const {
        return int64_t(pool_kind == 0 ? erec[0].bytes() : pool_kind == 1 ? brec[0].bytes() : frec[0].bytes());
    }

    // ---------------------------------------------------------------- GEMMs
    float *ws_for(bool hop) {
        if (sizing) return reinterpret_cast<float *>(uintptr_t(256));
        return hop ? ws_h.as<float>() : ws_c.as<float>();
    }

    template <int BNc, bool AMN, bool BMN, class Epi, int MODE>
    void run_pk(const char *name, double flops, const GemmPlan &gp, const typename Epi::Params &ep_in, cudaStream_t s,
                bool hop, int nh = 1, int nb = 1, int64_t out_bs = 0, int64_t out_hs = 0) {
        PkArgs a{};
        a.M = gp.args.M;
        a.N = gp.args.N;
        a.tiles_m = int(gp.grid.x);
        a.tiles_n = int(gp.grid.y);
        a.kb_per_seg = gp.args.kb_per_seg;
        a.n_seg = gp.args.n_seg;
        a.total_iters = a.kb_per_seg * a.n_seg;
        a.nbatch = nh * nb;
        a.nh = nh;
        a.out_bs = out_bs;
        a.out_hs = out_hs;
        const int tiles = a.tiles_m * a.tiles_n * a.nbatch;
        int splits = 1;
        if (MODE != GM_BATCH && tiles < sms()) splits = std::max(1, std::min(sms() / tiles, a.total_iters / split_min_kb()));
        a.iters_per_split = (a.total_iters + splits - 1) / splits;
        if (KIND == 1 && MODE != GM_BATCH) {
            // fp32 mode (as resnet_trainer.cu run_pk): every unit covers at most 256 of K inside one 3xTF32
            // segment, the partials summed in fp32 by pk_reduce_kernel in split order
            int ips = std::min(a.iters_per_split, std::min(a.kb_per_seg, 8));
            while (a.kb_per_seg % ips) --ips;
            a.iters_per_split = ips;
        }
        a.splits = (a.total_iters + a.iters_per_split - 1) / a.iters_per_split;
        using PL = PkLaunch<KIND, BNc, AMN, BMN, Epi, MODE>;
        a.units = tiles * a.splits;
        typename Epi::Params ep = a.splits > 1 ? Epi::for_split(ep_in) : ep_in;
        if constexpr (std::is_same<Epi, EpiConvOut2<KIND>>::value)
            if (a.splits > 1) ep.tiles = a.tiles_m * 4;
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
        L_(name, flops, 0.0, s, [&] { PL::launch(maps, a, ep, s, grid, paired); });
        if (a.splits > 1) {
            constexpr bool kStats = std::is_same<Epi, EpiConvOut2<KIND>>::value;
            constexpr int RC = kStats ? 32 : 16;  // rows per block: 256 threads x 2 float4 (stats) / 1 float4 (hop)
            constexpr int CC = 64;
            L_("splitk_reduce", 0, double(need) * 4, s, [&] {
                launch_pdl(pk_reduce_kernel<BNc, Epi, RC, CC>, dim3(tiles, 128 / RC, BNc / CC), dim3(256), 0, s, a,
                           ep);
            });
        }
    }

    static Operand opnd(const void *ptr, bool mn, int64_t mn_ext, int64_t k_ext, int64_t ld) {
        return Operand{ptr, mn, uint64_t(mn_ext), uint64_t(k_ext), uint64_t(ld)};
    }
    static COpnd copnd(const CBuf &b, bool mn, int64_t mn_ext, int64_t k_ext) {
        return COpnd{opnd(b.hi.p, mn, mn_ext, k_ext, b.ld), b.lo.p};
    }
    static COpnd copnd(const CTensor &t, bool mn, int64_t mn_ext, int64_t k_ext) {
        return COpnd{opnd(t.hi, mn, mn_ext, k_ext, t.ld), t.lo};
    }

    // D[M,N] = A . B with plain 2-D operands (bf16; fp32 mode: A.hi B.hi + A.hi B.lo + A.lo B.hi, 3xTF32).
    template <bool AMN, bool BMN, class Epi>
    void gemm(const char *name, const COpnd &A, const COpnd &Bo, int64_t M, int64_t N, int64_t Kd,
              const typename Epi::Params &ep, cudaStream_t s, bool hop) {
        Operand a[3] = {A.hi, A.hi, A.hi}, b[3] = {Bo.hi, Bo.hi, Bo.hi};
        const int nseg = KIND == 0 ? 1 : 3;
        b[1].ptr = Bo.lo;
        a[2].ptr = A.lo;
        bn_switch(tile_n(int(N)), [&](auto bnc) {
            constexpr int BNc = decltype(bnc)::value;
            if constexpr (BNc >= 64 && (KIND == 0 || BNc <= 128)) {
                GemmPlan p = plan_gemm<KIND, BNc, AMN, BMN>(a, b, nseg, int(M), int(N), int(Kd), 1, nullptr, nullptr);
                run_pk<BNc, AMN, BMN, Epi, GM_PLAIN>(name, 2.0 * M * N * Kd, p, ep, s, hop);
            } else {
                throw CdpError("unsupported GEMM tile width");
            }
        });
    }

    // ---------------------------------------------------------------- fused attention
    // 4-D TMA view {64 dims, T tokens, H heads, B samples} of a token-major bf16 buffer (row stride ld)
    CUtensorMap attn_map(const void *ptr, int64_t ld, int box_rows) const {
        const uint64_t dims[4] = {uint64_t(HD), uint64_t(T), uint64_t(H), uint64_t(B)};
        const uint64_t st[3] = {uint64_t(ld) * 2, uint64_t(HD) * 2, uint64_t(T) * ld * 2};
        const uint32_t box[4] = {64u, uint32_t(box_rows), 1u, 1u};
        const uint32_t es[4] = {1u, 1u, 1u, 1u};
        return make_tmap_4d(ptr, ElemType::BF16, dims, st, box, es, CU_TENSOR_MAP_SWIZZLE_128B);
    }
    AttnMaps attn_maps(const VRec &y) const {
        AttnMaps m;
        std::memset(&m, 0, sizeof(m));
        const int64_t qld = y.qkvb.ld;
        const __nv_bfloat16 *qkv = static_cast<const __nv_bfloat16 *>(y.qkvb.hi.p);
        m.q = attn_map(qkv, qld, 128);
        m.k = attn_map(qkv + D, qld, 256);
        m.v = attn_map(qkv + 2 * D, qld, 256);
        m.dout = attn_map(dattn.hi.p, dattn.ld, 128);
        return m;
    }
    AttnArgs attn_args(const VRec &y) const {
        AttnArgs a{};
        a.T = T;
        a.H = H;
        a.B = B;
        a.scale = 1.f / std::sqrt(float(HD));
        a.o = static_cast<__nv_bfloat16 *>(y.attn.hi.p);
        a.o_ld = y.attn.ld;
        a.lse = y.lse.as<float>();
        return a;
    }
    void attention_fwd(const VRec &y, cudaStream_t s) {
        const double tt = double(T) * T * HD * B * H;
        L_("attention", 4.0 * tt, double(R) * D * 2 * 4 + double(B) * H * T * 4, s, [&] {
            static bool attr = false;
            if (!attr) {
                CDP_CUDA(cudaFuncSetAttribute(attn_fwd_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                              kAttnFwdSmem));
                attr = true;
            }
            launch_pdl(attn_fwd_kernel, dim3(B * H * ((T + 127) / 128)), dim3(kAttnThreads), kAttnFwdSmem, s,
                       attn_maps(y), attn_args(y));
        });
    }
    void attention_bwd(const VRec &y, const CBuf &dqkv, cudaStream_t s) {
        const double tt = double(T) * T * HD * B * H;
        AttnArgs a = attn_args(y);
        a.dout = static_cast<const __nv_bfloat16 *>(dattn.hi.p);
        a.dout_ld = dattn.ld;
        a.dqkv = static_cast<__nv_bfloat16 *>(dqkv.hi.p);
        a.dqkv_ld = dqkv.ld;
        a.dk_off = D;
        a.dv_off = 2 * D;
        L_("attention_bwd", 10.0 * tt, double(R) * D * 2 * 8 + double(B) * H * T * 4, s, [&] {
            static bool attr = false;
            if (!attr) {
                CDP_CUDA(cudaFuncSetAttribute(attn_bwd_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                              kAttnBwdSmem));
                attr = true;
            }
            launch_pdl(attn_bwd_kernel, dim3(B * H), dim3(kAttnThreads), kAttnBwdSmem, s, attn_maps(y), a);
        });
    }

    // 4-D views of the token-major buffers: 64 columns from `col` of a [R][ld] buffer (per head: +64), and
    // the [B*H*T][ldp] probability-shaped buffers
    BView qview(const CBuf &b, int col) const {
        auto at = [&](const DevBuf &h) -> const void * {
            return h.p ? static_cast<const uint8_t *>(h.p) + size_t(col) * ES : nullptr;
        };
        return BView{at(b.hi), HD, T, b.ld, HD, int64_t(T) * b.ld, at(b.lo)};
    }
    BView pview(const CBuf &b) const {
        return BView{b.hi.p, T, T, b.ld, int64_t(T) * b.ld, int64_t(H) * T * b.ld, b.lo.p};
    }

    // Batched GEMM over (head, sample): operands are 4-D views {inner, rows, heads, samples}.
    template <bool AMN, bool BMN>
    void bgemm(const char *name, const BView &A, const BView &Bv, int M, int N, int K, void *out, int ld_out,
               int64_t out_bs, int64_t out_hs, int out_f32, cudaStream_t s, void *out_lo = nullptr) {
        bn_switch(tile_n(N), [&](auto bnc) {
            constexpr int BNc = decltype(bnc)::value;
            if constexpr (BNc >= 64 && (KIND == 0 || BNc <= 128)) {
                using Cfg = PkCfg<KIND, BNc, AMN, BMN, 0>;
                GemmPlan p{};
                std::memset(&p.maps, 0, sizeof(p.maps));
                auto mk = [&](const BView &v, const void *ptr, bool mn, int box_rows) {
                    const uint64_t dims[4] = {uint64_t(v.inner), uint64_t(v.rows), uint64_t(H), uint64_t(B)};
                    const uint64_t st[3] = {uint64_t(v.ld) * ES, uint64_t(v.hs) * ES, uint64_t(v.bs) * ES};
                    const uint32_t box[4] = {uint32_t(128 / ES), uint32_t(mn ? Cfg::BK : box_rows), 1u, 1u};
                    const uint32_t es[4] = {1u, 1u, 1u, 1u};
                    return make_tmap_4d(ptr, KIND == 0 ? ElemType::BF16 : ElemType::F32, dims, st, box, es,
                                        (KIND == 1 && mn) ? CU_TENSOR_MAP_SWIZZLE_128B_ATOM_32B
                                                          : CU_TENSOR_MAP_SWIZZLE_128B);
                };
                p.maps.a[0] = mk(A, A.ptr, AMN, 128);
                p.maps.b[0] = mk(Bv, Bv.ptr, BMN, BNc);
                if (KIND == 1) {  // 3xTF32: A.hi B.hi + A.hi B.lo + A.lo B.hi
                    p.maps.a[1] = p.maps.a[0];
                    p.maps.b[1] = mk(Bv, Bv.lo, BMN, BNc);
                    p.maps.a[2] = mk(A, A.lo, AMN, 128);
                    p.maps.b[2] = p.maps.b[0];
                }
                p.args.M = M;
                p.args.N = N;
                p.args.kb_per_seg = (K + Cfg::BK - 1) / Cfg::BK;
                p.args.n_seg = KIND == 0 ? 1 : 3;
                p.grid = dim3((M + 127) / 128, (N + BNc - 1) / BNc, 1);
                typename EpiConvOut2<KIND>::Params ep{};
                ep.out = out;
                ep.out_lo = out_lo;
                ep.ld = ld_out;
                ep.out_f32 = out_f32;
                run_pk<BNc, AMN, BMN, EpiConvOut2<KIND>, GM_BATCH>(name, 2.0 * M * N * K * H * B, p, ep, s, false, H, B,
                                                                 out_bs, out_hs);
            } else {
                throw CdpError("unsupported batched GEMM tile width");
            }
        });
    }

    // ---------------------------------------------------------------- plumbing
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
    // the worker that holds the complete gradient sum and runs the fused update
    bool is_updater() const { return W > 1 ? cw == W - 1 : rank == world - 1; }
    int wid() const { return W > 1 ? cw : rank; }  // worker index in trace records
    bool fresh_of(int unit) const { return W > 1 ? freshw[cw][unit] != 0 : units[unit].fresh != 0; }
    int vs(int unit, int p) const { return fresh_of(unit) ? p : (p ^ 1); }
    const float *th(int unit, int p) const { return theta[vs(unit, p)] + units[unit].base; }
    const CBuf &Wt(int unit, int p) const { return wc[vs(unit, p)][unit]; }
    const int *perm_w() const { return perm_dev.as<int>() + size_t(cw) * B; }
    void rec(int unit, int akind, int phase, int slot_, cudaStream_t s) {
        if (!trace) return;
        L_("trace_record", 0, 0, s, [&] {
            access_record_kernel<<<1, 1, 0, s>>>(TraceLog{tlog.as<uint32_t>(), tcur.as<uint32_t>(), kTraceCap}, ring,
                                                 wid(), unit + 1, akind, phase, slot_,
                                                 (const int *)&ctrl_dev.as<Control>()->step);
            CDP_CUDA(cudaGetLastError());
        });
    }
    // forward (A_FWD) / backward (A_BWD) read of `units` around `f` (trace mode)
    template <class F>
    void reading(std::initializer_list<int> us, int akind, int p, cudaStream_t s, F &&f) {
        for (int u : us) rec(u, akind, 0, vs(u, p), s);
        f();
        for (int u : us) rec(u, akind, 1, vs(u, p), s);
    }
    template <class F>
    void traced_update(int unit, int p, bool updates, cudaStream_t s, F &&launch) {
        if (updates) rec(unit, A_UPD, 0, p, s);
        launch();
        if (trace && updates) {
            L_("trace_vtag", 0, 0, s, [&] {
                vtag_update_kernel<<<1, 1, 0, s>>>(ring, unit + 1, (const int *)&ctrl_dev.as<Control>()->step);
                CDP_CUDA(cudaGetLastError());
            });
            rec(unit, A_NEW, 1, p ^ 1, s);
        }
    }
    // live-record accounting (W > 1): the executed high-water mark of activation-record bytes
    void live_delta(int pool_kind, int sign) {
        if (!probe) return;
        const int64_t d = sign * record_bytes(pool_kind);
        L_("live_probe", 0, 0, cs, [&] {
            live_probe_kernel<<<1, 1, 0, cs>>>(live.as<int64_t>(), d);
            CDP_CUDA(cudaGetLastError());
        });
    }

    HopParams hop_params(int unit, int p) {
        const VUnit &u = units[unit];
        HopParams hp{};
        if (W > 1)  // one GPU: the chain w1 -> ... -> wW runs in plan order on the hop stream
            hp.mode = cw == 0 ? 0 : cw == W - 1 ? 2 : 1;
        else
            hp.mode = world == 1 ? 3 : (rank == 0 ? 0 : rank == world - 1 ? 2 : 1);
        hp.stage = unit + 1;
        hp.base = u.base;
        hp.din = u.rows;
        hp.dout = u.cols;
        hp.s_in = (W == 1 && rank > 0) ? prev_partial : partial;
        hp.s_out = partial;
        hp.theta_cur = theta[p];
        hp.theta_new = theta[p ^ 1];
        hp.vel = vel;
        hp.lr = &ctrl_dev.as<Control>()->lr;
        hp.momentum = momentum;
        hp.wd = wd;
        hp.n_mb = float(W > 1 ? W : world);
        hp.wc_new = u.kind == V_LIN ? wc[p ^ 1][unit].view() : CTensor{};
        Flags *fl = flags_dev.as<Flags>();
        hp.grad_flags = &fl->grad;
        hp.upd_flags = &fl->upd;
        hp.sync.enabled = W == 1 ? 1 : 0;
        hp.sync.n_readers = chain.empty() ? world - 1 : 1;  // pull chain: only its head takes from the updater
        hp.sync.step = &ctrl_dev.as<Control>()->step;
        hp.sync.own = ring;
        hp.sync.prev = prev_ring;
        hp.sync.cta_counter = cta_counters.as<unsigned>();
        hp.sync.pre_external = 1;
        return hp;
    }
    void hop_wait(const HopParams &hp, cudaStream_t s) {
        if (world == 1 || W > 1 || hp.mode >= 3) return;
        L_("hop_wait", 0, 0, s, [&] {
            hop_wait_kernel<<<1, 128, 0, s>>>(hp);
            CDP_CUDA(cudaGetLastError());
        });
    }
    void pull(int unit, int p, cudaStream_t s) {
        if (W > 1 || rank == world - 1 || world == 1 || sizing) return;
        const VUnit &u = units[unit];
        const int vslot = vs(unit, p);
        CTensor w = u.kind == V_LIN ? wc[vslot][unit].view() : CTensor{};
        if (!chain.empty()) {  // forwarding along the reader order (rank_common.cuh chain kernels)
            const int st = u.stage - 1, pr = chain[size_t(st) * 2], sc = chain[size_t(st) * 2 + 1];
            RingFlags *pf = pr < 0 ? upd_ring : reinterpret_cast<RingFlags *>(peer_regions[pr]);
            const float *src = (pr < 0 ? upd_theta[vslot]
                                       : reinterpret_cast<const float *>(peer_regions[pr] + region_off) + vslot * Pp) +
                               u.base;
            L_("pull_wait", 0, 0, s, [&] {
                chain_wait_kernel<<<1, 32, 0, s>>>(pf, pr < 0 ? 1 : 0, ring, unit + 1, u.fresh, sc >= 0 ? 1 : 0,
                                                   (const int *)&ctrl_dev.as<Control>()->step);
                CDP_CUDA(cudaGetLastError());
            });
            L_("pull", 0, double(u.n) * 10, s, [&] {
                launch_pdl(chain_pull_kernel<KIND>, dim3(blocks_for(u.n, 1024)), dim3(256), 0, s, src,
                           theta[vslot] + u.base, u.n, std::max(u.cols, 1), w, pf, pr < 0 ? 1 : 0, ring, unit + 1,
                           u.fresh, (const int *)&ctrl_dev.as<Control>()->step,
                           cta_counters.as<unsigned>() + kMaxStages, trace ? 1 : 0);
            });
            return;
        }
        L_("pull_wait", 0, 0, s, [&] {
            pull_wait_kernel<<<1, 32, 0, s>>>(upd_ring, ring, unit + 1, u.fresh,
                                              (const int *)&ctrl_dev.as<Control>()->step);
            CDP_CUDA(cudaGetLastError());
        });
        L_("pull", 0, double(u.n) * 10, s, [&] {
            launch_pdl(pull_tensor_kernel<KIND>, dim3(blocks_for(u.n, 1024)), dim3(256), 0, s,
                       (const float *)(upd_theta[vslot] + u.base), theta[vslot] + u.base, u.n, std::max(u.cols, 1),
                       w, upd_ring, ring, unit + 1, u.fresh, (const int *)&ctrl_dev.as<Control>()->step,
                       cta_counters.as<unsigned>() + kMaxStages, trace ? 1 : 0);
        });
    }

    // Weight gradient of a linear unit fused with its hop / update: [A, 1]^T . dY on the hop stream.
    void lin_hop(int unit, int p, const CTensor &a_in, int64_t krows, const CTensor &dy, cudaEvent_t dy_ready,
                 cudaEvent_t dgrad_done) {
        const VUnit &u = units[unit];
        wait(hs, dy_ready);
        if (dgrad_done && !fresh_of(unit) && is_updater()) wait(hs, dgrad_done);
        HopParams hp = hop_params(unit, p);
        hop_wait(hp, hs);
        traced_update(unit, p, hp.mode >= 2, hs, [&] {
            gemm<true, true, EpiHop2<KIND>>("lin_wgrad_hop", copnd(a_in, true, u.rows, krows),
                                         copnd(dy, true, u.cols, krows), u.rows, u.cols, krows, hp, hs, true);
        });
    }
    void ln_hop(int unit, int p, const float *dg, const float *db, cudaEvent_t ready) {
        wait(hs, ready);
        HopParams hp = hop_params(unit, p);
        hop_wait(hp, hs);
        traced_update(unit, p, hp.mode >= 2, hs, [&] {
            L_("ln_hop", 0, double(D) * 2 * 24, hs, [&] {
                launch_pdl(vector_hop_kernel, dim3(1), dim3(128), 0, hs, hp, dg, db, D);
            });
        });
    }

    // ---------------------------------------------------------------- layers
    void layernorm(const float *x, int rows, int stride, int unit, int p, const CTensor &out, float *mean,
                   float *rstd, cudaStream_t s) {
        reading({unit}, A_FWD, p, s, [&] { layernorm_(x, rows, stride, unit, p, out, mean, rstd, s); });
    }
    void layernorm_(const float *x, int rows, int stride, int unit, int p, const CTensor &out, float *mean,
                    float *rstd, cudaStream_t s) {
        auto go = [&](auto kern) {
            L_("ln_fwd", 0, double(rows) * D * 6, s, [&] {
                launch_pdl(kern, dim3((rows * 32 + 255) / 256), dim3(256), 0, s, x, rows, stride, D, th(unit, p), eps,
                           out, mean, rstd);
            });
        };
        switch (D % 128 == 0 ? D / 128 : 0) {  // row in registers as 16-byte columns
            case 1: go(ln_fwd4_kernel<KIND, 1>); break;
            case 2: go(ln_fwd4_kernel<KIND, 2>); break;
            case 4: go(ln_fwd4_kernel<KIND, 4>); break;
            case 6: go(ln_fwd4_kernel<KIND, 6>); break;
            case 8: go(ln_fwd4_kernel<KIND, 8>); break;
            default: go(ln_fwd_kernel<KIND>); break;
        }
    }
    // LayerNorm backward of `unit`: dh_out = dh_in + LN'(g); parameter gradients -> dgam / dbet.
    void layernorm_bwd(const float *g, const float *x, int rows, int stride, int unit, int p, const float *mean,
                       const float *rstd, const float *dh_in, float *dh_out, float *dgam, float *dbet,
                       cudaStream_t s, CTensor copy = CTensor{}) {
        reading({unit}, A_BWD, p, s, [&] {
            layernorm_bwd_(g, x, rows, stride, unit, p, mean, rstd, dh_in, dh_out, dgam, dbet, s, copy);
        });
    }
    void layernorm_bwd_(const float *g, const float *x, int rows, int stride, int unit, int p, const float *mean,
                        const float *rstd, const float *dh_in, float *dh_out, float *dgam, float *dbet,
                        cudaStream_t s, CTensor copy) {
        const int rpc = ln_bwd_rows();
        const int nblk = (rows + rpc - 1) / rpc;
        const size_t smem = size_t(8) * D * 2 * 4;
        auto go = [&](auto kern) {
            if (!ln_attr_) {
                CDP_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem)));
            }
            L_("ln_bwd", 0, double(rows) * D * (16 + (copy.hi ? 2 : 0)), s, [&] {
                launch_pdl(kern, dim3(nblk), dim3(256), smem, s, g, x, rows, stride, D, th(unit, p), mean, rstd,
                           dh_in, dh_out, copy, lnpart.as<double>(), rpc);
            });
        };
        switch (D % 128 == 0 ? D / 128 : 0) {  // 16-byte columns
            case 1: go(ln_bwd_fused4_kernel<KIND, 1>); break;
            case 2: go(ln_bwd_fused4_kernel<KIND, 2>); break;
            case 4: go(ln_bwd_fused4_kernel<KIND, 4>); break;
            case 6: go(ln_bwd_fused4_kernel<KIND, 6>); break;
            case 8: go(ln_bwd_fused4_kernel<KIND, 8>); break;
            default:
                switch (D / 32) {
                    case 2: go(ln_bwd_fused_kernel<KIND, 2>); break;
                    default: throw CdpError("LayerNorm width must be 64, 128, 256, 512, 768 or 1024");
                }
        }
        ln_attr_ = !sizing;
        L_("ln_param_finalize", 0, double(nblk) * D * 16, s, [&] {
            launch_pdl(bn_finalize_bwd_kernel, dim3((D * 32 + 255) / 256), dim3(256), 0, s,
                       (const double *)lnpart.as<double>(), nblk, D, dbet, dgam);
        });
    }
    bool ln_attr_ = false;

    // ---------------------------------------------------------------- segments (forward)
    ERec &erec_w() { return erec[slot[cw][0]]; }
    VRec &brec_w(int l) { return brec[slot[cw][1 + l]]; }
    FRec &frec_w() { return frec[slot[cw][L + 1]]; }

    // embedding: patches -> tokens (+ class token, position embedding) into block 0's record
    void fwd_embed(int p, cudaStream_t s) {
        live_delta(0, +1);
        live_delta(L > 0 ? 1 : 2, +1);
        pull(u_patch, p, s);
        pull(u_cls, p, s);
        pull(u_pos, p, s);
        const int K0 = P * P * 3;
        CBuf &patches = erec_w().patches;
        L_("patch_im2col", 0, double(B) * NP * patches.ld * 2, s, [&] {
            launch_pdl(patch_im2col_kernel<KIND>, dim3(blocks_for(int64_t(B) * NP * patches.ld)), dim3(256), 0, s,
                       (const float *)data_x.as<float>(), perm_w(), img, P, G, B * NP, patches.view());
        });
        {
            typename EpiConvOut2<KIND>::Params ep{};
            ep.out = E.p;
            ep.ld = D;
            ep.out_f32 = 1;
            const CBuf &w = Wt(u_patch, p);
            reading({u_patch}, A_FWD, p, s, [&] {
                gemm<false, true, EpiConvOut2<KIND>>("patch_embed", copnd(patches, false, B * NP, K0 + 1),
                                                  copnd(w, true, D, K0 + 1), B * NP, D, K0 + 1, ep, s, false);
            });
        }
        float *h0 = L > 0 ? brec_w(0).h.template as<float>() : frec_w().hL.template as<float>();
        reading({u_cls, u_pos}, A_FWD, p, s, [&] {
            L_("embed_assemble", 0, double(R) * D * 12, s, [&] {
                launch_pdl(embed_assemble_kernel, dim3(blocks_for(int64_t(R) * D)), dim3(256), 0, s,
                           (const float *)E.as<float>(), th(u_cls, p), th(u_pos, p), B, T, D, h0);
            });
        });
    }

    void fwd_block(int l, int p, cudaStream_t s) {
        const VBlock &b = blocks[l];
        VRec &y = brec_w(l);
        live_delta(l + 1 < L ? 1 : 2, +1);
        float *hout = l + 1 < L ? brec_w(l + 1).h.template as<float>() : frec_w().hL.template as<float>();
        for (int u : {b.ln1, b.qkv, b.proj, b.ln2, b.fc1, b.fc2}) pull(u, p, s);
        layernorm(y.h.as<float>(), R, 1, b.ln1, p, y.u1.view(), y.m1.as<float>(), y.r1.as<float>(), s);
        {
            typename EpiConvOut2<KIND>::Params ep{};
            ep.out = y.qkvb.hi.p;
            ep.out_lo = y.qkvb.lo.p;
            ep.ld = y.qkvb.ld;
            const CBuf &w = Wt(b.qkv, p);
            reading({b.qkv}, A_FWD, p, s, [&] {
                gemm<false, true, EpiConvOut2<KIND>>("qkv", copnd(y.u1, false, R, D + 1),
                                                  copnd(w, true, 3 * D, D + 1), R, 3 * D, D + 1, ep, s,
                                                  false);
            });
        }
        // attention: S = Q K^T (fp32) -> P = softmax(scale S) (bf16) -> O = P V
        const float scale = 1.f / std::sqrt(float(HD));
        const int64_t qld = y.qkvb.ld;
        const BView Q = qview(y.qkvb, 0), Kv = qview(y.qkvb, D), V = qview(y.qkvb, 2 * D);
        const BView Pv = pview(y.P);
        if (fused_attn) {
            attention_fwd(y, s);
        } else {
        bgemm<false, false>("attn_scores", Q, Kv, T, T, HD, S.p, lds, int64_t(H) * T * lds, int64_t(T) * lds, 1, s);
        L_("softmax", 0, double(B) * H * T * T * 6, s, [&] {
            const dim3 g((B * H * T * 32 + 255) / 256);
            const float *Sp = S.as<float>();
            __nv_bfloat16 *Pp = y.P.hi.as<__nv_bfloat16>();
            if (KIND == 1)
                launch_pdl(softmax_fwd_c_kernel<KIND>, g, dim3(256), 0, s, Sp, B * H * T, T, lds, scale, y.P.view());
            else if (T <= 128)
                launch_pdl(softmax_fwd4_kernel<1>, g, dim3(256), 0, s, Sp, B * H * T, T, lds, scale, Pp, ldp);
            else if (T <= 256)
                launch_pdl(softmax_fwd4_kernel<2>, g, dim3(256), 0, s, Sp, B * H * T, T, lds, scale, Pp, ldp);
            else
                launch_pdl(softmax_fwd_kernel, g, dim3(256), 0, s, Sp, B * H * T, T, lds, scale, Pp, ldp);
        });
        bgemm<false, true>("attn_values", Pv, V, T, HD, T, y.attn.hi.p, y.attn.ld, int64_t(T) * y.attn.ld, HD, 0, s,
                           y.attn.lo.p);
        }
        {
            typename EpiConvOut2<KIND>::Params ep{};
            ep.out = y.hmid.p;
            ep.ld = D;
            ep.out_f32 = 1;
            ep.add = y.h.p;
            const CBuf &w = Wt(b.proj, p);
            reading({b.proj}, A_FWD, p, s, [&] {
                gemm<false, true, EpiConvOut2<KIND>>("proj", copnd(y.attn, false, R, D + 1),
                                                  copnd(w, true, D, D + 1), R, D, D + 1, ep, s, false);
            });
        }
        layernorm(y.hmid.as<float>(), R, 1, b.ln2, p, y.u2.view(), y.m2.as<float>(), y.r2.as<float>(), s);
        {
            typename EpiConvOut2<KIND>::Params ep{};
            ep.out = y.z1.hi.p;  // gelu'(z) (the backward's factor), not z
            ep.ld = y.z1.ld;
            ep.gelu_out = y.g1.view();
            ep.out_gelu_grad = 1;
            const CBuf &w = Wt(b.fc1, p);
            reading({b.fc1}, A_FWD, p, s, [&] {
                gemm<false, true, EpiConvOut2<KIND>>("fc1_gelu", copnd(y.u2, false, R, D + 1),
                                                  copnd(w, true, F, D + 1), R, F, D + 1, ep, s, false);
            });
        }
        {
            typename EpiConvOut2<KIND>::Params ep{};
            ep.out = hout;
            ep.ld = D;
            ep.out_f32 = 1;
            ep.add = y.hmid.p;
            const CBuf &w = Wt(b.fc2, p);
            reading({b.fc2}, A_FWD, p, s, [&] {
                gemm<false, true, EpiConvOut2<KIND>>("fc2", copnd(y.g1, false, R, F + 1),
                                                  copnd(w, true, D, F + 1), R, D, F + 1, ep, s, false);
            });
        }
    }

    // final LayerNorm + head on the class token, loss -> dz and this worker's loss slot
    void fwd_final(int p, cudaStream_t s) {
        FRec &f = frec_w();
        pull(u_ln, p, s);
        pull(u_head, p, s);
        layernorm(f.hL.as<float>(), B, T, u_ln, p, f.uf.view(), f.mf.as<float>(), f.rf.as<float>(), s);
        {
            typename EpiConvOut2<KIND>::Params ep{};
            ep.out = f.z.p;
            ep.ld = classes;
            ep.out_f32 = 1;
            const CBuf &w = Wt(u_head, p);
            reading({u_head}, A_FWD, p, s, [&] {
                gemm<false, true, EpiConvOut2<KIND>>("head", copnd(f.uf, false, B, D + 1),
                                                  copnd(w, true, classes, D + 1), B, classes, D + 1, ep, s,
                                                  false);
            });
        }
        Flags *fl = flags_dev.as<Flags>();
        double *lw = loss_w.as<double>() + cw;
        const int nt = std::max(32, round_up(B, 32));
        const size_t lsm = sizeof(double) * nt + sizeof(float) * B * classes;
        if (classes <= 64 && lsm <= 48 * 1024) {
            L_("loss", 0, 0, s, [&] {
                launch_pdl(loss_kernel<KIND>, dim3(1), dim3(nt), lsm, s, (const float *)f.z.as<float>(), B, classes,
                           loss_kind, perm_w(), (const int *)data_lab.as<int>(), (const float *)nullptr, f.dz.view(),
                           lw, &fl->loss);
            });
        } else {
            L_("loss", 0, 0, s, [&] {
                launch_pdl(xent_rows_kernel<KIND>, dim3(B), dim3(256), 0, s, (const float *)f.z.as<float>(), B, classes,
                           perm_w(), (const int *)data_lab.as<int>(), f.dz.view(), loss_rows.as<double>());
            });
            L_("loss_sum", 0, 0, s, [&] {
                launch_pdl(loss_sum_kernel, dim3(1), dim3(1), 0, s, (const double *)loss_rows.as<double>(), B, lw,
                           &fl->loss);
            });
        }
    }

    // ---------------------------------------------------------------- segments (backward)
    void bwd_final(int p) {
        FRec &f = frec_w();
        VCarry &c = carry[cw];
        cudaEvent_t dz_ready = ev(cs);
        {
            typename EpiConvOut2<KIND>::Params ep{};
            ep.out = duf.p;
            ep.ld = D;
            ep.out_f32 = 1;
            const CBuf &w = Wt(u_head, p);
            reading({u_head}, A_BWD, p, cs, [&] {
                gemm<false, false, EpiConvOut2<KIND>>("head_dgrad", copnd(f.dz, false, B, classes),
                                                   copnd(w, false, D, classes), B, D, classes, ep, cs, false);
            });
        }
        cudaEvent_t head_dg = ev(cs);
        lin_hop(u_head, p, f.uf.view(), B, f.dz.view(), dz_ready, head_dg);
        // final LayerNorm (class-token rows only): dh = 0 elsewhere (and its bf16 copy, the last block's operand)
        const CBuf *out_c = L > 0 ? &dhc(L - 1) : nullptr;
        if (!sizing) {
            CDP_CUDA(cudaMemsetAsync(c.dh.p, 0, c.dh.bytes, cs));
            if (out_c) CDP_CUDA(cudaMemsetAsync(out_c->hi.p, 0, out_c->hi.bytes, cs));
            if (out_c && out_c->lo.p) CDP_CUDA(cudaMemsetAsync(out_c->lo.p, 0, out_c->lo.bytes, cs));
        }
        layernorm_bwd(duf.as<float>(), f.hL.as<float>(), B, T, u_ln, p, f.mf.as<float>(), f.rf.as<float>(), nullptr,
                      c.dh.as<float>(), dgf.as<float>(), dbf.as<float>(), cs, out_c ? out_c->view() : CTensor{});
        ln_hop(u_ln, p, dgf.as<float>(), dbf.as<float>(), ev(cs));
        live_delta(2, -1);
    }

    void bwd_block(int l, int p) {
        const VBlock &b = blocks[l];
        VRec &y = brec_w(l);
        VGrad &gr = grad_of(l);
        VCarry &c = carry[cw];
        float *dh = c.dh.as<float>();
        const CBuf &dhc_in = dhc(l);
        const float scale = 1.f / std::sqrt(float(HD));
        // ---- MLP (dhc_in = bf16(dh), written by the LayerNorm backward that produced dh)
        cudaEvent_t dhc_ready = ev(cs);
        {
            typename EpiConvOut2<KIND>::Params ep{};
            ep.out = gr.dz1.hi.p;
            ep.out_lo = gr.dz1.lo.p;
            ep.ld = gr.dz1.ld;
            ep.mul = y.z1.hi.p;  // stored gelu'(z)
            const CBuf &w = Wt(b.fc2, p);
            // the factor rows TMA-staged into shared memory by warp 3, the product stored by TMA (EpiConvAddT)
            static const bool staged = std::getenv("CDP_NO_TMA_ADD") == nullptr;
            reading({b.fc2}, A_BWD, p, cs, [&] {
                if constexpr (KIND == 0) {
                    if (staged && EpiConvAddT<KIND>::eligible(ep, F, tile_n(F)) && tile_n(F) >= 128) {
                        gemm<false, false, EpiConvAddT<KIND>>("fc2_dgrad_gelu", copnd(dhc_in, false, R, D),
                                                              copnd(w, false, F, D), R, F, D, ep, cs, false);
                        return;
                    }
                }
                gemm<false, false, EpiConvOut2<KIND>>("fc2_dgrad_gelu", copnd(dhc_in, false, R, D),
                                                      copnd(w, false, F, D), R, F, D, ep, cs, false);
            });
        }
        cudaEvent_t dz1_ready = ev(cs);
        lin_hop(b.fc2, p, y.g1.view(), R, dhc_in.view(), dhc_ready, dz1_ready);
        {
            typename EpiConvOut2<KIND>::Params ep{};
            ep.out = du.p;
            ep.ld = D;
            ep.out_f32 = 1;
            const CBuf &w = Wt(b.fc1, p);
            reading({b.fc1}, A_BWD, p, cs, [&] {
                gemm<false, false, EpiConvOut2<KIND>>("fc1_dgrad", copnd(gr.dz1, false, R, F),
                                                   copnd(w, false, D, F), R, D, F, ep, cs, false);
            });
        }
        cudaEvent_t fc1_dg = ev(cs);
        lin_hop(b.fc1, p, y.u2.view(), R, gr.dz1.view(), dz1_ready, fc1_dg);
        layernorm_bwd(du.as<float>(), y.hmid.as<float>(), R, 1, b.ln2, p, y.m2.as<float>(), y.r2.as<float>(), dh,
                      dhm.as<float>(), gr.dg2.as<float>(), gr.db2.as<float>(), cs, gr.dhmc.view());
        ln_hop(b.ln2, p, gr.dg2.as<float>(), gr.db2.as<float>(), ev(cs));
        // ---- attention
        cudaEvent_t dhmc_ready = ev(cs);
        {
            typename EpiConvOut2<KIND>::Params ep{};
            ep.out = dattn.hi.p;
            ep.out_lo = dattn.lo.p;
            ep.ld = dattn.ld;
            const CBuf &w = Wt(b.proj, p);
            reading({b.proj}, A_BWD, p, cs, [&] {
                gemm<false, false, EpiConvOut2<KIND>>("proj_dgrad", copnd(gr.dhmc, false, R, D),
                                                   copnd(w, false, D, D), R, D, D, ep, cs, false);
            });
        }
        cudaEvent_t proj_dg = ev(cs);
        lin_hop(b.proj, p, y.attn.view(), R, gr.dhmc.view(), dhmc_ready, proj_dg);
        const int64_t qld = y.qkvb.ld;
        auto qv = [&](int col) { return qview(y.qkvb, col); };
        const int64_t dld = gr.dqkv.ld;
        if (fused_attn) {
            attention_bwd(y, gr.dqkv, cs);
        } else {
        const BView dO = qview(dattn, 0);
        const BView Pv = pview(y.P);
        const BView dSv = pview(dS);
        bgemm<false, false>("attn_dprobs", dO, qv(2 * D), T, T, HD, dP.p, lds, int64_t(H) * T * lds, int64_t(T) * lds,
                            1, cs);
        L_("softmax_bwd", 0, double(B) * H * T * T * 8, cs, [&] {
            const dim3 g((B * H * T * 32 + 255) / 256);
            const float *dPp = dP.as<float>();
            const __nv_bfloat16 *Pp = y.P.hi.as<__nv_bfloat16>();
            __nv_bfloat16 *dSp = static_cast<__nv_bfloat16 *>(dS.hi.p);
            if (KIND == 1)
                launch_pdl(softmax_bwd_c_kernel<KIND>, g, dim3(256), 0, cs, dPp, y.P.view(), B * H * T, T, lds, scale,
                           dS.view());
            else if (T <= 128)
                launch_pdl(softmax_bwd4_kernel<1>, g, dim3(256), 0, cs, dPp, Pp, B * H * T, T, lds, ldp, scale, dSp);
            else if (T <= 256)
                launch_pdl(softmax_bwd4_kernel<2>, g, dim3(256), 0, cs, dPp, Pp, B * H * T, T, lds, ldp, scale, dSp);
            else
                launch_pdl(softmax_bwd_kernel, g, dim3(256), 0, cs, dPp, Pp, B * H * T, T, lds, ldp, scale, dSp);
        });
        auto dq = [&](const DevBuf &half, int col) -> void * {
            return half.p ? static_cast<uint8_t *>(half.p) + size_t(col) * ES : nullptr;
        };
        bgemm<true, true>("attn_dvalues", Pv, dO, T, HD, T, dq(gr.dqkv.hi, 2 * D), int(dld), int64_t(T) * dld, HD, 0,
                          cs, dq(gr.dqkv.lo, 2 * D));
        bgemm<false, true>("attn_dquery", dSv, qv(D), T, HD, T, dq(gr.dqkv.hi, 0), int(dld), int64_t(T) * dld, HD, 0,
                           cs, dq(gr.dqkv.lo, 0));
        bgemm<true, true>("attn_dkey", dSv, qv(0), T, HD, T, dq(gr.dqkv.hi, D), int(dld), int64_t(T) * dld, HD, 0, cs,
                          dq(gr.dqkv.lo, D));
        }
        cudaEvent_t dqkv_ready = ev(cs);
        {
            typename EpiConvOut2<KIND>::Params ep{};
            ep.out = du.p;
            ep.ld = D;
            ep.out_f32 = 1;
            const CBuf &w = Wt(b.qkv, p);
            reading({b.qkv}, A_BWD, p, cs, [&] {
                gemm<false, false, EpiConvOut2<KIND>>("qkv_dgrad", copnd(gr.dqkv, false, R, 3 * D),
                                                   copnd(w, false, D, 3 * D), R, D, 3 * D, ep, cs, false);
            });
        }
        cudaEvent_t qkv_dg = ev(cs);
        lin_hop(b.qkv, p, y.u1.view(), R, gr.dqkv.view(), dqkv_ready, qkv_dg);
        layernorm_bwd(du.as<float>(), y.h.as<float>(), R, 1, b.ln1, p, y.m1.as<float>(), y.r1.as<float>(),
                      dhm.as<float>(), dh, gr.dg1.as<float>(), gr.db1.as<float>(), cs,
                      l > 0 ? dhc(l - 1).view() : CTensor{});
        ln_hop(b.ln1, p, gr.dg1.as<float>(), gr.db1.as<float>(), ev(cs));
        live_delta(1, -1);
    }

    void bwd_embed(int p) {
        const float *dh = carry[cw].dh.as<float>();
        L_("token_grad", 0, double(R) * D * 4, cs, [&] {
            launch_pdl(token_grad_kernel, dim3(blocks_for(int64_t(T) * D)), dim3(256), 0, cs, dh, B, T, D,
                       gpos.as<float>(), gcls.as<float>());
        });
        cast(dh, B * NP, NP, T, 1, dE.view(), cs);
        cudaEvent_t emb_ready = ev(cs);
        wait(hs, emb_ready);
        for (int u : {u_pos, u_cls}) {
            HopParams hp = hop_params(u, p);
            hop_wait(hp, hs);
            const float *g = u == u_pos ? gpos.as<float>() : gcls.as<float>();
            traced_update(u, p, hp.mode >= 2, hs, [&] {
                L_("vec_hop", 0, double(units[u].n) * 24, hs, [&] {
                    launch_pdl(flat_hop_kernel, dim3(blocks_for(units[u].n, 1024)), dim3(256), 0, hs, hp, g,
                               units[u].n);
                });
            });
        }
        lin_hop(u_patch, p, erec_w().patches.view(), B * NP, dE.view(), emb_ready, nullptr);
        live_delta(0, -1);
    }

    void cast(const float *in, int rows, int per, int in_per, int skip, const CTensor &out, cudaStream_t s) {
        L_("cast", 0, double(rows) * D * 6, s, [&] {
            launch_pdl(cast_rows_kernel<KIND>, dim3(blocks_for(int64_t(rows) * D)), dim3(256), 0, s, in, rows, D, per,
                       in_per, skip, out);
        });
    }

    void fwd_seg(int s, int p) {
        if (s == 0) fwd_embed(p, cs);
        else if (s <= L) fwd_block(s - 1, p, cs);
        else fwd_final(p, cs);
    }
    void bwd_seg(int s, int p) {
        if (s == 0) bwd_embed(p);
        else if (s <= L) bwd_block(s - 1, p);
        else bwd_final(p);
    }

    // One training step of every worker this process runs.  W == 1 (one worker per GPU): forward over
    // all segments, backward in reverse, weight gradients + hops on the hop stream lagging the compute
    // stream.  W > 1 (single-GPU cyclic CDP): the plan's F / B tasks in timeline order (ref
    // schedule.py:236-257), each expanded into its segments; the hop stream is joined before every
    // segment, so per-block backward operands and released record slots are never overwritten while a
    // weight gradient still reads them, and the gradient chain S = g_1 + ... + g_W runs in worker order.
    void record_step(int p) {
        kernels_per_step = 0;
        flops_per_step = 0.0;
        cudaEvent_t fork = ev(main);
        wait(cs, fork);
        wait(hs, fork);
        if (W == 1) {
            cw = 0;
            for (int s = 0; s <= L + 1; ++s) fwd_seg(s, p);
            for (int s = L + 1; s >= 0; --s) bwd_seg(s, p);
        } else {
            for (const VOp &op : plan) {
                cw = op.worker - 1;
                std::vector<int> segs;
                for (int s = 0; s <= L + 1; ++s)
                    if (seg_stage[s] == op.stage) segs.push_back(s);
                if (op.kind == 1) std::reverse(segs.begin(), segs.end());
                for (int s : segs) {
                    wait(cs, ev(hs));
                    if (op.kind == 0)
                        fwd_seg(s, p);
                    else
                        bwd_seg(s, p);
                }
            }
        }
        // join + bookkeeping
        wait(main, ev(cs));
        wait(main, ev(hs));
        L_("loss_mean", 0, 0, main, [&] {
            loss_mean_kernel<<<1, 1, 0, main>>>(loss_w.as<double>(), W, loss_dev.as<double>());
            CDP_CUDA(cudaGetLastError());
        });
        L_("finish_step", 0, 0, main, [&] {
            finish_step_kernel_rn<<<1, 1, 0, main>>>(loss_dev.as<double>(), flags_dev.as<Flags>(),
                                                     hist_loss.as<double>(), hist_flags.as<Flags>(), hist_cap,
                                                     &ctrl_dev.as<Control>()->step);
            CDP_CUDA(cudaGetLastError());
        });
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
                record_step(p);
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
    void pack_slot(int sl) {
        for (size_t i = 0; i < units.size(); ++i) {
            const VUnit &u = units[i];
            if (u.kind != V_LIN) continue;
            pack_tensor_kernel<KIND><<<blocks_for(u.n), 256, 0, main>>>(theta[sl] + u.base, u.n, u.cols,
                                                                     wc[sl][i].view());
            CDP_CUDA(cudaGetLastError());
        }
    }
    void set_params(int which, const float *host) {
        for (int v = 0; v < 2; ++v) {
            if (which >= 0 && v != which) continue;
            const int sl = v == 0 ? (t & 1) : ((t & 1) ^ 1);
            CDP_CUDA(cudaMemcpyAsync(theta[sl], host, size_t(Pn) * 4, cudaMemcpyHostToDevice, main));
            pack_slot(sl);
            std::vector<uint32_t> tag(kMaxStages, uint32_t(v == 0 ? t : t - 1));  // version tags (ref engine.py:8-10)
            CDP_CUDA(cudaMemcpy(ring->vtag[sl], tag.data(), kMaxStages * 4, cudaMemcpyHostToDevice));
        }
        CDP_CUDA(cudaStreamSynchronize(main));
    }
    void get_params(int which, float *host) {
        CDP_CUDA(cudaStreamSynchronize(main));
        const int slot = which == 0 ? (t & 1) : ((t & 1) ^ 1);
        CDP_CUDA(cudaMemcpy(host, theta[slot], size_t(Pn) * 4, cudaMemcpyDeviceToHost));
    }
    void stage_control(const int *perm, float lr) {
        const int k = stage_next;
        stage_next = (stage_next + 1) % RING_N;
        CDP_CUDA(cudaEventSynchronize(stage_ev[k]));
        uint8_t *blk = stage_host + size_t(k) * stage_bytes;
        Control *c = reinterpret_cast<Control *>(blk);
        c->lr = lr;
        c->step = t;
        std::memcpy(blk + sizeof(Control), perm, size_t(W) * B * 4);
        CDP_CUDA(cudaMemcpyAsync(ctrl_dev.p, blk, sizeof(Control), cudaMemcpyHostToDevice, main));
        CDP_CUDA(cudaMemcpyAsync(perm_dev.p, blk + sizeof(Control), size_t(W) * B * 4, cudaMemcpyHostToDevice, main));
        CDP_CUDA(cudaEventRecord(stage_ev[k], main));
    }
    void step(const int *perm, float lr) {
        stage_control(perm, lr);
        CDP_CUDA(cudaGraphLaunch(exec[t & 1], main));
        ++t;
    }
    void step_host_batch(const float *x, const int32_t *labels, float lr) {
        const size_t im = size_t(img) * img * 3;
        const int n = W * B;  // every worker's micro-batch, worker-major
        CDP_CUDA(cudaMemcpyAsync(data_x.p, x, size_t(n) * im * 4, cudaMemcpyHostToDevice, main));
        CDP_CUDA(cudaMemcpyAsync(data_lab.p, labels, size_t(n) * 4, cudaMemcpyHostToDevice, main));
        std::vector<int> ident(n);
        for (int i = 0; i < n; ++i) ident[i] = i;
        step(ident.data(), lr);
    }
    void profile_step(const int *perm, float lr, bool serial) {
        stage_control(perm, lr);
        clear_oprecs();
        instr = true;
        cudaStream_t sc = cs, sh = hs;
        if (serial) cs = hs = main;
        try {
            record_step(t & 1);
        } catch (...) {
            instr = false;
            cs = sc;
            hs = sh;
            throw;
        }
        cs = sc;
        hs = sh;
        instr = false;
        ++t;
        CDP_CUDA(cudaDeviceSynchronize());
    }
};

}  // namespace cdp

using namespace cdp;

struct cdp_vit {
    std::unique_ptr<VitTrainer<0>> b16;  // bf16 operands
    std::unique_ptr<VitTrainer<1>> f32;  // fp32 mode
};

// run fn on the trainer of either mode (C-ABI entry points), errors as cdp status codes
template <class Fn>
static int with_vit(cdp_vit *tr, Fn &&fn) {
    return guarded([&] {
        CDP_REQUIRE(tr && (tr->b16 || tr->f32), "null ViT trainer");
        if (tr->b16)
            fn(*tr->b16);
        else
            fn(*tr->f32);
    });
}

template <int KIND>
static std::unique_ptr<VitTrainer<KIND>> vit_new(int image, int patch, int dim, int depth, int heads, int mlp, int classes,
                                           int micro_batch, int workers, float momentum, float weight_decay,
                                           int n_samples, const float *x, const int32_t *labels) {
    CDP_REQUIRE(micro_batch >= 1 && micro_batch <= 256, "micro-batch must be in [1, 256]");
    CDP_REQUIRE(depth >= 1 && depth <= 40, "depth: 1..40");
    auto tr = std::make_unique<VitTrainer<KIND>>();
    tr->B = micro_batch;
    tr->img = image;
    tr->P = patch;
    tr->D = dim;
    tr->L = depth;
    tr->H = heads;
    tr->F = mlp;
    tr->classes = classes;
    tr->momentum = momentum;
    tr->wd = weight_decay;
    tr->W = workers;
    tr->n_samples = std::max(n_samples, micro_batch * workers);
    const size_t im = size_t(image) * image * 3;
    tr->data_x = DevBuf(size_t(tr->n_samples) * im * 4);
    tr->data_lab = DevBuf(size_t(tr->n_samples) * 4);
    if (x) CDP_CUDA(cudaMemcpy(tr->data_x.p, x, size_t(n_samples) * im * 4, cudaMemcpyHostToDevice));
    if (labels) CDP_CUDA(cudaMemcpy(tr->data_lab.p, labels, size_t(n_samples) * 4, cudaMemcpyHostToDevice));
    tr->make_units();
    return tr;
}

extern "C" int cdp_vit_create_rank(int image, int patch, int dim, int depth, int heads, int mlp, int classes,
                                   int micro_batch, int world, int rank, const int32_t *unit_stage,
                                   const uint8_t *stage_fresh, float momentum, float weight_decay, int n_samples,
                                   const float *x, const int32_t *labels, int dtype, cdp_vit **out) {
    return guarded([&] {
        CDP_REQUIRE(world >= 1 && rank >= 0 && rank < world, "bad rank / world");
        CDP_REQUIRE(dtype == CDP_DTYPE_BF16 || dtype == CDP_DTYPE_FP32, "dtype: CDP_DTYPE_BF16 or CDP_DTYPE_FP32");
        auto make = [&](auto kind) {
        auto tr = vit_new<decltype(kind)::value>(image, patch, dim, depth, heads, mlp, classes, micro_batch, 1,
                                                 momentum, weight_decay, n_samples, x, labels);
        tr->rank = rank;
        tr->world = world;
        for (size_t i = 0; i < tr->units.size(); ++i) {
            const int st = unit_stage[i];
            CDP_REQUIRE(st >= 1 && st <= world, "unit stage out of range");
            tr->units[i].stage = st;
            tr->units[i].fresh = stage_fresh[st - 1] != 0;
        }
        // one worker: every block keeps its own record (embed / final: one each)
        tr->slot.assign(1, std::vector<int>(size_t(depth) + 2, 0));
        for (int l = 0; l < depth; ++l) tr->slot[0][1 + l] = l;
        tr->pool[1] = depth;
        tr->build();
        return tr;
        };
        std::unique_ptr<cdp_vit> h(new cdp_vit{});
        if (dtype == CDP_DTYPE_BF16)
            h->b16 = make(std::integral_constant<int, 0>{});
        else
            h->f32 = make(std::integral_constant<int, 1>{});
        *out = h.release();
    });
}

extern "C" int cdp_vit_create_cyclic(int image, int patch, int dim, int depth, int heads, int mlp, int classes,
                                     int micro_batch, int n_workers, const int32_t *unit_stage, const uint8_t *fresh,
                                     int n_ops, const int32_t *ops, const int32_t *rec_slot, const int32_t *pools,
                                     float momentum, float weight_decay, int probe, int n_samples, const float *x,
                                     const int32_t *labels, int dtype, cdp_vit **out) {
    return guarded([&] {
        CDP_REQUIRE(n_workers >= 2, "single-GPU cyclic CDP needs at least two workers (micro-batches)");
        CDP_REQUIRE(dtype == CDP_DTYPE_BF16 || dtype == CDP_DTYPE_FP32, "dtype: CDP_DTYPE_BF16 or CDP_DTYPE_FP32");
        auto make = [&](auto kind) {
        auto tr = vit_new<decltype(kind)::value>(image, patch, dim, depth, heads, mlp, classes, micro_batch,
                                                 n_workers, momentum, weight_decay, n_samples, x, labels);
        const int NS = depth + 2;
        tr->seg_stage.assign(NS, 0);
        for (size_t i = 0; i < tr->units.size(); ++i) {
            const int st = unit_stage[i];
            CDP_REQUIRE(st >= 1 && st <= n_workers, "unit stage out of range");
            tr->units[i].stage = st;
            int &ss = tr->seg_stage[tr->seg_of_unit(int(i))];
            CDP_REQUIRE(ss == 0 || ss == st, "the units of an embedding / block / head segment must share a stage");
            ss = st;
        }
        tr->freshw.assign(n_workers, std::vector<uint8_t>(tr->units.size(), 1));
        for (int w = 0; w < n_workers; ++w)
            for (size_t i = 0; i < tr->units.size(); ++i)
                tr->freshw[w][i] = fresh[size_t(w) * n_workers + tr->units[i].stage - 1] != 0;
        std::vector<int> f_seen(n_workers, 0), b_seen(n_workers, 0);
        for (int k = 0; k < n_ops; ++k) {
            const VOp op{ops[3 * k], ops[3 * k + 1], ops[3 * k + 2]};
            CDP_REQUIRE((op.kind == 0 || op.kind == 1) && op.worker >= 1 && op.worker <= n_workers && op.stage >= 1 &&
                            op.stage <= n_workers,
                        "bad plan op");
            ++(op.kind ? b_seen : f_seen)[op.worker - 1];
            tr->plan.push_back(op);
        }
        for (int w = 0; w < n_workers; ++w)
            CDP_REQUIRE(f_seen[w] == n_workers && b_seen[w] == n_workers, "the plan must hold every F / B task once");
        for (int k = 0; k < 3; ++k) {
            CDP_REQUIRE(pools[k] >= 1, "record pools need at least one slot");
            tr->pool[k] = pools[k];
        }
        tr->slot.assign(n_workers, std::vector<int>(NS, 0));
        for (int w = 0; w < n_workers; ++w)
            for (int sg = 0; sg < NS; ++sg) {
                const int v = rec_slot[size_t(w) * NS + sg];
                const int k = sg == 0 ? 0 : sg <= depth ? 1 : 2;
                CDP_REQUIRE(v >= 0 && v < pools[k], "record slot out of range");
                tr->slot[w][sg] = v;
            }
        tr->probe = probe != 0;
        tr->build();
        return tr;
        };
        std::unique_ptr<cdp_vit> h(new cdp_vit{});
        if (dtype == CDP_DTYPE_BF16)
            h->b16 = make(std::integral_constant<int, 0>{});
        else
            h->f32 = make(std::integral_constant<int, 1>{});
        *out = h.release();
    });
}

extern "C" int cdp_vit_set_trace(cdp_vit *tr, int on) {
    return with_vit(tr, [&](auto &m) {
        CDP_REQUIRE(!m.exec[0], "set the trace option before cdp_vit_connect (it changes the captured step)");
        m.trace = on != 0;
        if (m.trace && !m.tlog.p) {
            m.tlog = DevBuf(size_t(std::decay_t<decltype(m)>::kTraceCap) * kTraceWords * 4);
            m.tcur = DevBuf(4);
        }
    });
}

extern "C" int cdp_vit_trace(cdp_vit *tr, uint32_t *records, int max_records, int *count) {
    return with_vit(tr, [&](auto &m) {
        CDP_REQUIRE(m.trace, "trace option not set");
        CDP_CUDA(cudaStreamSynchronize(m.main));
        uint32_t n = 0;
        CDP_CUDA(cudaMemcpy(&n, m.tcur.p, 4, cudaMemcpyDeviceToHost));
        CDP_REQUIRE(n <= std::decay_t<decltype(m)>::kTraceCap, "trace buffer overflow: read the records more often");
        *count = int(n);
        const int k = std::min<int>(int(n), max_records);
        if (k > 0) CDP_CUDA(cudaMemcpy(records, m.tlog.p, size_t(k) * kTraceWords * 4, cudaMemcpyDeviceToHost));
        CDP_CUDA(cudaMemset(m.tcur.p, 0, 4));
    });
}

extern "C" int cdp_vit_info(cdp_vit *tr, int64_t *n_params, int *n_units) {
    return with_vit(tr, [&](auto &m) {
        *n_params = m.Pn;
        *n_units = int(m.units.size());
    });
}

extern "C" int cdp_vit_region(cdp_vit *tr, void **base) {
    return with_vit(tr, [&](auto &m) { *base = m.region.p; });
}

extern "C" int cdp_vit_ipc_handle(cdp_vit *tr, void *handle64) {
    return with_vit(tr, [&](auto &m) {
        cudaIpcMemHandle_t h;
        CDP_CUDA(cudaIpcGetMemHandle(&h, m.region.p));
        std::memcpy(handle64, &h, sizeof(h));
    });
}

extern "C" int cdp_vit_pull_chain(cdp_vit *tr, const int32_t *pred_succ, int n_stages) {
    return with_vit(tr, [&](auto &m) {
        CDP_REQUIRE(!m.exec[0], "the pull chain is set before connect (graph capture)");
        CDP_REQUIRE(n_stages == 0 || (n_stages == m.world && pred_succ), "pull chain: one row per stage");
        for (int k = 0; k < 2 * n_stages; ++k)
            CDP_REQUIRE(pred_succ[k] >= -1 && pred_succ[k] < m.world - 1 && pred_succ[k] != m.rank,
                        "pull chain: ranks of other readers");
        m.chain.assign(pred_succ, pred_succ + size_t(n_stages) * 2);
    });
}

extern "C" int cdp_vit_connect(cdp_vit *tr, void *const *regions) {
    return with_vit(tr, [&](auto &m) {
        auto at = [&](int r) { return static_cast<uint8_t *>(regions[r]); };
        if (m.rank > 0) {
            m.prev_ring = reinterpret_cast<RingFlags *>(at(m.rank - 1));
            m.prev_partial = reinterpret_cast<float *>(at(m.rank - 1) + m.region_off) + 2 * m.Pp;
        }
        const int u = m.world - 1;
        m.upd_ring = reinterpret_cast<RingFlags *>(at(u));
        m.upd_theta[0] = reinterpret_cast<float *>(at(u) + m.region_off);
        m.upd_theta[1] = m.upd_theta[0] + m.Pp;
        m.peer_regions.assign(size_t(m.world), nullptr);
        for (int r = 0; r < m.world; ++r) m.peer_regions[r] = at(r);
        m.capture();
    });
}

extern "C" void cdp_vit_destroy(cdp_vit *tr) {
    if (tr) {
        cudaDeviceSynchronize();
        delete tr;
    }
}

extern "C" int cdp_vit_set_params(cdp_vit *tr, int which, const float *theta) {
    return with_vit(tr, [&](auto &m) { m.set_params(which, theta); });
}

extern "C" int cdp_vit_get_params(cdp_vit *tr, int which, float *theta) {
    return with_vit(tr, [&](auto &m) { m.get_params(which, theta); });
}

extern "C" int cdp_vit_step(cdp_vit *tr, const int32_t *perm, float lr) {
    return with_vit(tr, [&](auto &m) { m.step(perm, lr); });
}

extern "C" int cdp_vit_step_host_batch(cdp_vit *tr, const float *x, const int32_t *labels, float lr) {
    return with_vit(tr, [&](auto &m) { m.step_host_batch(x, labels, lr); });
}

extern "C" int cdp_vit_profile_step(cdp_vit *tr, const int32_t *perm, float lr, int serial, int max_ops, char *names,
                                    int name_len, double *flops, double *bytes, float *ms, int *n_ops) {
    return with_vit(tr, [&](auto &m) {
        m.profile_step(perm, lr, serial != 0);
        const int n = std::min<int>(max_ops, int(m.oprecs.size()));
        *n_ops = int(m.oprecs.size());
        for (int i = 0; i < n; ++i) {
            const auto &o = m.oprecs[i];
            std::strncpy(names + size_t(i) * name_len, o.name.c_str(), name_len - 1);
            names[size_t(i) * name_len + name_len - 1] = 0;
            flops[i] = o.flops;
            bytes[i] = o.bytes;
            CDP_CUDA(cudaEventElapsedTime(&ms[i], o.a, o.b));
        }
    });
}

extern "C" int cdp_vit_history(cdp_vit *tr, int max, double *losses, uint32_t *flags, int *count) {
    return with_vit(tr, [&](auto &m) {
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

extern "C" int cdp_vit_sync(cdp_vit *tr) {
    return with_vit(tr, [&](auto &m) { CDP_CUDA(cudaStreamSynchronize(m.main)); });
}

extern "C" int cdp_vit_ring_error(cdp_vit *tr, int *err) {
    return with_vit(tr, [&](auto &m) {
        CDP_CUDA(cudaStreamSynchronize(m.main));
        uint32_t e = 0;
        CDP_CUDA(cudaMemcpy(&e, &m.ring->err, 4, cudaMemcpyDeviceToHost));
        *err = int(e);
    });
}

extern "C" int cdp_vit_stats(cdp_vit *tr, int64_t *out, int n_out) {
    // [0] activation-record bytes allocated (record pools: embed / block / final slots x record bytes),
    // [1] parameter-state bytes, [2] kernels / step, [3] tensor-core flops / step,
    // [4] executed high-water mark of live record bytes (probe; 0 when off),
    // [5..7] bytes of one embed / block / final record, [8..10] slots per pool
    return with_vit(tr, [&](auto &m) {
        int64_t act = 0;
        for (int k = 0; k < 3; ++k) act += m.record_bytes(k) * m.pool[k];
        int64_t par = int64_t(m.Pp) * (m.vel ? 16 : 12);
        for (int v = 0; v < 2; ++v)
            for (auto &w : m.wc[v]) par += int64_t(cbytes(w));
        int64_t hw[2] = {0, 0};
        if (m.probe) {
            CDP_CUDA(cudaStreamSynchronize(m.main));
            CDP_CUDA(cudaMemcpy(hw, m.live.p, 16, cudaMemcpyDeviceToHost));
        }
        int64_t vals[11] = {act, par, m.kernels_per_step, int64_t(m.flops_per_step), hw[1], m.record_bytes(0),
                            m.record_bytes(1), m.record_bytes(2), m.pool[0], m.pool[1], m.pool[2]};
        for (int i = 0; i < n_out && i < 11; ++i) out[i] = vals[i];
    });
}

extern "C" int cdp_vit_mark(cdp_vit *tr, int k) {
    return with_vit(tr, [&](auto &m) {
        while (int(m.marks.size()) <= k) {
            cudaEvent_t e;
            CDP_CUDA(cudaEventCreate(&e));
            m.marks.push_back(e);
        }
        CDP_CUDA(cudaEventRecord(m.marks[k], m.main));
    });
}

extern "C" int cdp_vit_elapsed(cdp_vit *tr, int a, int b, float *ms) {
    return with_vit(tr, [&](auto &m) {
        CDP_CUDA(cudaEventSynchronize(m.marks[b]));
        CDP_CUDA(cudaEventElapsedTime(ms, m.marks[a], m.marks[b]));
    });
}

extern "C" int cdp_vit_flush_l2(cdp_vit *tr) {
    return with_vit(tr, [&](auto &m) {
        if (!m.flush_buf.p) m.flush_buf = DevBuf(size_t(256) << 20);
        CDP_CUDA(cudaMemsetAsync(m.flush_buf.p, m.t & 0xff, m.flush_buf.bytes, m.main));
    });
}

// Fused attention on caller-owned device buffers (tests / tools): forward O = softmax(Q K^T / 8) V and
// the row log-sum-exp; with backward != 0 also dQ, dK, dV from dO into dqkv (Q | K | V column blocks
// of width H * 64, like qkv).  Synchronous.
extern "C" int cdp_attention(const void *qkv, int64_t qkv_ld, const void *dout, int64_t dout_ld, int T, int H, int B,
                             void *o, int64_t o_ld, float *lse, void *dqkv, int64_t dqkv_ld, int backward) {
    using namespace cdp;
    return guarded([&] {
        CDP_REQUIRE(T >= 1 && T <= 256 && H >= 1 && B >= 1, "fused attention: 1 <= T <= 256");
        CDP_REQUIRE(qkv_ld % 8 == 0 && o_ld % 8 == 0 && (!backward || (dout_ld % 8 == 0 && dqkv_ld % 8 == 0)),
                    "row strides must be multiples of 8 elements");
        const int64_t D = int64_t(H) * 64;
        auto map = [&](const void *ptr, int64_t ld, int rows) {
            const uint64_t dims[4] = {64u, uint64_t(T), uint64_t(H), uint64_t(B)};
            const uint64_t st[3] = {uint64_t(ld) * 2, 128u, uint64_t(T) * ld * 2};
            const uint32_t box[4] = {64u, uint32_t(rows), 1u, 1u};
            const uint32_t es[4] = {1u, 1u, 1u, 1u};
            return make_tmap_4d(ptr, ElemType::BF16, dims, st, box, es, CU_TENSOR_MAP_SWIZZLE_128B);
        };
        AttnMaps m;
        std::memset(&m, 0, sizeof(m));
        const __nv_bfloat16 *q = static_cast<const __nv_bfloat16 *>(qkv);
        m.q = map(q, qkv_ld, 128);
        m.k = map(q + D, qkv_ld, 256);
        m.v = map(q + 2 * D, qkv_ld, 256);
        if (backward) m.dout = map(dout, dout_ld, 128);
        AttnArgs a{};
        a.T = T;
        a.H = H;
        a.B = B;
        a.scale = 0.125f;
        a.o = static_cast<__nv_bfloat16 *>(o);
        a.o_ld = o_ld;
        a.lse = lse;
        CDP_CUDA(cudaFuncSetAttribute(attn_fwd_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, kAttnFwdSmem));
        attn_fwd_kernel<<<B * H * ((T + 127) / 128), kAttnThreads, kAttnFwdSmem>>>(m, a);
        CDP_CUDA(cudaGetLastError());
        if (backward) {
            a.dout = static_cast<const __nv_bfloat16 *>(dout);
            a.dout_ld = dout_ld;
            a.dqkv = static_cast<__nv_bfloat16 *>(dqkv);
            a.dqkv_ld = dqkv_ld;
            a.dk_off = D;
            a.dv_off = 2 * D;
            CDP_CUDA(cudaFuncSetAttribute(attn_bwd_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, kAttnBwdSmem));
            attn_bwd_kernel<<<B * H, kAttnThreads, kAttnBwdSmem>>>(m, a);
            CDP_CUDA(cudaGetLastError());
        }
        CDP_CUDA(cudaDeviceSynchronize());
    });
}
