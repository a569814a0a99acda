// Device-resident CDP / DP training step for the stage-stacked MLP.
//
// Replaces the reference's `_advance` (training/engine.py:66-116) end to end:
// per-(micro-batch, stage) version selection, per-micro-batch value+grad
// (training/_kernels.pyx:25-132), ascending-i gradient accumulation and the
// SGD(+momentum) update.  Execution follows a step plan compiled from the
// reference-parity Timeline (paper_2403_08837_b200/executor.py):
//   * one CUDA stream per worker; F/B tasks of worker i are launched in its
//     plan order; cross-worker edges (ring-hop order, activation-slot reuse)
//     become event edges;
//   * each B task = [loss kernel] -> dgrad GEMM (fused tanh', bias grad) ->
//     wgrad GEMM whose epilogue IS the gradient hop S_i = S_{i-1} + g_i and,
//     on the last worker, the SGD update writing version t+1;
//   * the whole step is captured once per version parity into a CUDA graph.
// Parameter versions live in two slots (slot = version mod 2); the update of
// step t writes slot (t+1) mod 2, which only held version t-1.
#include <cuda_bf16.h>

#include <algorithm>
#include <array>
#include <cstring>
#include <map>
#include <memory>
#include <mutex>
#include <tuple>
#include <vector>

#include "../../include/cdp_b200.h"
#include "gemm_launch.cuh"
#include "mlp_kernels.cuh"
#include "trainer_common.cuh"

namespace cdp {

enum OpField { OP_KIND = 0, OP_WORKER, OP_STAGE, OP_FRESH, OP_REC_IN, OP_REC_OUT, OP_HOP, OP_FIELDS_PAD, OP_FIELDS };
enum HopMode { HOP_FIRST = 0, HOP_MID = 1, HOP_LAST = 2, HOP_ONLY = 3, HOP_GRAD = 4 };

struct StageGeom {
    int din, dout;
    int64_t base;
};

// -------------------------------------------------------------------------
struct MlpTrainer {
    int kind = 0;  // 0 bf16, 1 fp32 (3xTF32)
    int S = 0, W = 0, B = 0, loss_kind = 1;
    float momentum = 0.f, wd = 0.f;
    std::vector<StageGeom> st;
    int64_t P = 0;
    int n_samples = 0;
    int dmax = 0;

    // plan
    std::vector<std::array<int, OP_FIELDS>> ops;
    std::vector<std::pair<int, int>> deps;
    std::vector<int> slots;  // per stage (1..S) number of input-record slots

    // device state
    // IPC-shareable region: [RingFlags | theta slot 0 | theta slot 1 | partial S]
    DevBuf region, vel;
    float *theta[2] = {nullptr, nullptr};
    float *partial = nullptr;
    RingFlags *ring = nullptr;
    size_t region_theta_off = 0;
    int64_t Pp = 0;  // padded slot stride (floats)
    // multi-GPU (one process per GPU): this rank's global worker index and peers
    int rank = -1, world = 1;
    RingFlags *prev_ring = nullptr;      // rank - 1
    float *prev_partial = nullptr;
    RingFlags *upd_ring = nullptr;       // updater = rank world - 1
    float *upd_theta[2] = {nullptr, nullptr};
    DevBuf cta_counters;                 // [2][kMaxStages]: hop / pull launches
    std::vector<CBuf> wc[2];                  // [slot][stage]
    std::vector<std::vector<CBuf>> rec;       // [stage][slot]
    DevBuf loss_all;  // [W] per-worker micro-batch losses (double)
    struct Worker {
        DevBuf z, ws, counters;
        double *loss = nullptr;
        std::vector<CBuf> dz;  // per layer: dZ_l [B][dout_l] (written once per step)
        cudaStream_t stream = nullptr;   // compute chain: pulls, forward, loss, data gradients
        cudaStream_t hstream = nullptr;  // gradient hops: weight-grad GEMMs + fused hop / update
    };
    std::vector<Worker> wk;
    DevBuf data_x, data_lab, data_tgt;
    DevBuf ctrl_dev, perm_dev, flags_dev, hist_loss, hist_flags, hist_count;
    // ring of pinned host staging blocks {Control, perm}: a block is reused only
    // after the H2D copy that read it has executed (event), so back-to-back
    // asynchronous steps never see a later step's permutation or lr
    static constexpr int RING = 16;
    uint8_t *stage_host = nullptr;
    size_t stage_bytes = 0;
    cudaEvent_t stage_ev[RING] = {};
    int stage_next = 0;
    int hist_cap = 1 << 14;
    size_t ws_floats = 0;

    cudaStream_t main = nullptr;
    std::vector<cudaEvent_t> op_events, hop_events, loss_events;
    cudaEvent_t fork_ev = nullptr;
    std::vector<cudaEvent_t> join_ev;
    cudaGraphExec_t exec[2] = {nullptr, nullptr};
    int t = 1;  // training step of the next launch; current version = t
    int kernels_per_step = 0;
    int launch_mask = 7;  // bit0 gather/loss, bit1 fwd/dgrad GEMM, bit2 wgrad(+hop) GEMM
    bool trace = false;   // stamp %globaltimer around every op (executed-schedule export)
    DevBuf trace_buf;     // [n_ops][4] u64: compute start, compute end, hop start, hop end
    std::vector<cudaEvent_t> marks;
    DevBuf flush_buf;

    ~MlpTrainer() {
        for (auto &e : exec)
            if (e) cudaGraphExecDestroy(e);
        for (auto e : op_events) cudaEventDestroy(e);
        for (auto e : hop_events) cudaEventDestroy(e);
        for (auto e : loss_events) cudaEventDestroy(e);
        for (auto e : join_ev) cudaEventDestroy(e);
        if (fork_ev) cudaEventDestroy(fork_ev);
        for (auto &w : wk) {
            if (w.stream) cudaStreamDestroy(w.stream);
            if (w.hstream) cudaStreamDestroy(w.hstream);
        }
        if (main) cudaStreamDestroy(main);
        for (auto e : stage_ev)
            if (e) cudaEventDestroy(e);
        for (auto e : marks) cudaEventDestroy(e);
        if (stage_host) cudaFreeHost(stage_host);
    }

    // ---------------------------------------------------------------- GEMM sizing
    int bn_rows(int) const { return 32; }  // narrow N tiles: more CTAs for the latency-bound small GEMMs
    int bn_mn(int n) const {  // MN-major B tile width
        const int ch = kind == 0 ? 64 : 32;
        return std::min(256, round_up(std::max(std::min(n, 64), ch), ch));
    }
    int splits_for(int M, int N, int BN, int K, bool allow_split = true) const {
        if (!allow_split) return 1;
        const int bk = kind == 0 ? 64 : 32;
        const int nseg = kind == 0 ? 1 : 3;
        const int kb = (K + bk - 1) / bk;
        const int total = kb * nseg;
        const int tiles = ((M + 127) / 128) * ((N + BN - 1) / BN);
        int s = std::max(1, std::min(total, 16 / std::max(tiles, 1)));
        if (kind == 1) s = std::max(s, (total + 7) / 8);  // <= 256 of K per TMEM accumulation
        s = std::min(s, total);
        const int per = (total + s - 1) / s;
        return (total + per - 1) / per;
    }
    size_t ws_need(int M, int N, int BN, int K) const {
        const int s = splits_for(M, N, BN, K);
        if (s <= 1) return 0;
        return size_t((M + 127) / 128) * ((N + BN - 1) / BN) * s * 128 * BN;
    }

    // ---------------------------------------------------------------- setup
    void setup(const int64_t *dims, int n_dims) {
        S = n_dims - 1;
        CDP_REQUIRE(S >= 1, "dims needs at least input and output widths");
        CDP_REQUIRE(S <= kMaxStages, "too many layers");
        CDP_REQUIRE(B >= 1 && B <= 256, "micro-batch size must be in [1, 256]");
        int64_t off = 0;
        for (int j = 0; j < S; ++j) {
            StageGeom g{int(dims[j]), int(dims[j + 1]), off};
            CDP_REQUIRE(g.din >= 1 && g.dout >= 1, "layer widths must be positive");
            off += int64_t(g.din) * g.dout + g.dout;
            st.push_back(g);
            dmax = std::max({dmax, g.din, g.dout});
        }
        P = off;
        for (int v = 0; v < 2; ++v) {
            for (int j = 0; j < S; ++j) wc[v].push_back(make_cbuf(kind, st[j].din + 1, st[j].dout));
        }
        if (momentum != 0.f) vel = DevBuf(size_t(P) * 4);
        region_theta_off = (sizeof(RingFlags) + 255) / 256 * 256;
        Pp = (P + 63) / 64 * 64;  // slot stride keeps every slot 256-byte aligned
        region = DevBuf(region_theta_off + size_t(Pp) * 4 * 3);
        ring = region.as<RingFlags>();
        theta[0] = reinterpret_cast<float *>(region.as<uint8_t>() + region_theta_off);
        theta[1] = theta[0] + Pp;
        partial = theta[1] + Pp;
        cta_counters = DevBuf(2 * kMaxStages * 4);
        rec.resize(S);
        for (int j = 0; j < S; ++j)
            for (int r = 0; r < std::max(1, slots[j + 1]); ++r) {
                rec[j].push_back(make_cbuf(kind, B, st[j].din + 1));
                if (kind == 0)
                    ones_column_kernel<0><<<1, 256>>>(rec[j].back().view(), B, st[j].din);
                else
                    ones_column_kernel<1><<<1, 256>>>(rec[j].back().view(), B, st[j].din);
                CDP_CUDA(cudaGetLastError());
            }
        // split-K workspace: the largest need of any GEMM a worker runs
        for (int j = 0; j < S; ++j) {
            ws_floats = std::max(ws_floats, ws_need(st[j].dout, B, bn_rows(B), st[j].din + 1));
            ws_floats = std::max(ws_floats, ws_need(st[j].din, B, bn_rows(B), st[j].dout));
        }
        wk.resize(W);
        loss_all = DevBuf(size_t(W) * 8);
        for (int i = 0; i < W; ++i) wk[i].loss = loss_all.as<double>() + i;
        for (auto &w : wk) {
            w.z = DevBuf(size_t(B) * st[S - 1].dout * 4);
            w.ws = DevBuf(std::max<size_t>(ws_floats, 1) * 4);
            w.counters = DevBuf(4096 * 4);
            for (int j = 0; j < S; ++j) w.dz.push_back(make_cbuf(kind, B, st[j].dout));
            CDP_CUDA(cudaStreamCreateWithFlags(&w.stream, cudaStreamNonBlocking));
            CDP_CUDA(cudaStreamCreateWithFlags(&w.hstream, cudaStreamNonBlocking));
        }
        CDP_CUDA(cudaStreamCreateWithFlags(&main, cudaStreamNonBlocking));
        ctrl_dev = DevBuf(sizeof(Control));
        perm_dev = DevBuf(size_t(W) * B * 4);
        flags_dev = DevBuf(sizeof(Flags));
        hist_loss = DevBuf(size_t(hist_cap) * 8);
        hist_flags = DevBuf(size_t(hist_cap) * sizeof(Flags));
        hist_count = DevBuf(4);
        stage_bytes = (sizeof(Control) + size_t(W) * B * 4 + 255) / 256 * 256;
        CDP_CUDA(cudaMallocHost(&stage_host, stage_bytes * RING));
        for (auto &e : stage_ev) CDP_CUDA(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
    }

    void upload_data(int n, const float *x, const int *labels, const float *targets) {
        n_samples = std::max(n, W * B);
        data_x = DevBuf(size_t(n_samples) * st[0].din * 4);
        if (x) CDP_CUDA(cudaMemcpy(data_x.p, x, size_t(n) * st[0].din * 4, cudaMemcpyHostToDevice));
        if (loss_kind == 1) {
            data_lab = DevBuf(size_t(n_samples) * 4);
            if (labels) CDP_CUDA(cudaMemcpy(data_lab.p, labels, size_t(n) * 4, cudaMemcpyHostToDevice));
        } else {
            data_tgt = DevBuf(size_t(n_samples) * st[S - 1].dout * 4);
            if (targets)
                CDP_CUDA(cudaMemcpy(data_tgt.p, targets, size_t(n) * st[S - 1].dout * 4, cudaMemcpyHostToDevice));
        }
    }

    // ---------------------------------------------------------------- GEMM launches
    template <int K>
    static Operand op_of(const CBuf &b, bool lo, bool mn_major, int mn, int k) {
        return Operand{lo ? b.lo.p : b.hi.p, mn_major, uint64_t(mn), uint64_t(k), uint64_t(b.ld)};
    }

    // Segments for (A, B): bf16 1; 3xTF32 (hi,hi), (hi,lo), (lo,hi).
    template <int K>
    static int segments(const CBuf &a, bool amn, int am, int ak, const CBuf &b, bool bmn, int bn_, int bk,
                        Operand *A, Operand *Bo) {
        if (K == 0) {
            A[0] = op_of<K>(a, false, amn, am, ak);
            Bo[0] = op_of<K>(b, false, bmn, bn_, bk);
            return 1;
        }
        A[0] = op_of<K>(a, false, amn, am, ak), Bo[0] = op_of<K>(b, false, bmn, bn_, bk);
        A[1] = op_of<K>(a, false, amn, am, ak), Bo[1] = op_of<K>(b, true, bmn, bn_, bk);
        A[2] = op_of<K>(a, true, amn, am, ak), Bo[2] = op_of<K>(b, false, bmn, bn_, bk);
        return 3;
    }

    template <int K, bool AMN, bool BMN, class Epi>
    void gemm(int BN, const Operand *A, const Operand *Bo, int nseg, int M, int N, int Kd, Worker &w,
              const typename Epi::Params &ep, cudaStream_t s) {
        const int splits = splits_for(M, N, BN, Kd, !Epi::kTile);
        GemmPlan p;
#define CDP_GEMM_BN(BN_)                                                                                            \
    case BN_:                                                                                                       \
        if constexpr ((!BMN || BN_ % (K == 0 ? 64 : 32) == 0) && (!Epi::kTile || BN_ <= 64)) {                    \
            p = plan_gemm<K, BN_, AMN, BMN>(A, Bo, nseg, M, N, Kd, splits, w.ws.as<float>(), w.counters.as<int>()); \
            CDP_REQUIRE(gemm_ws_floats(p, BN_) <= ws_floats, "split-K workspace too small");                      \
            launch_gemm<K, BN_, AMN, BMN, Epi>(p, ep, s);                                                          \
            ++kernels_per_step;                                                                                    \
            return;                                                                                                \
        }                                                                                                           \
        break;
        switch (BN) {
            CDP_GEMM_BN(32)
            CDP_GEMM_BN(64)
            CDP_GEMM_BN(128)
            CDP_GEMM_BN(256)
            default:
                break;
        }
#undef CDP_GEMM_BN
        throw CdpError("unsupported GEMM tile width " + std::to_string(BN));
    }

    // ---------------------------------------------------------------- tasks
    template <int K>
    void forward(int w, int j, int vslot, int rin, int rout, cudaStream_t s, const int *perm_w) {
        const StageGeom &g = st[j];
        Worker &wr = wk[w];
        if (j == 0 && (launch_mask & 1)) {
            launch_pdl(gather_kernel<K>, dim3(B), dim3(256), 0, s, (const float *)data_x.as<float>(), g.din, perm_w,
                       rec[0][rin].view());
            ++kernels_per_step;
        }
        Operand A[3], Bo[3];
        // z = [h, 1] . [W; b]: K = din + 1 folds the bias into the product
        const int nseg =
            segments<K>(wc[vslot][j], true, g.dout, g.din + 1, rec[j][rin], false, B, g.din + 1, A, Bo);
        typename EpiFwd<K>::Params ep{};
        ep.last = j == S - 1;
        if (ep.last)
            ep.z = wr.z.as<float>();
        else
            ep.out = rec[j + 1][rout].view();
        if (launch_mask & 2) gemm<K, true, false, EpiFwd<K>>(bn_rows(B), A, Bo, nseg, g.dout, B, g.din + 1, wr, ep, s);
    }

    // B task, compute half: [loss] then the data gradient dZ_{j-1} (W rows only).
    template <int K>
    void bwd_compute(int w, int j, int vslot, int rin, cudaStream_t s, const int *perm_w, cudaEvent_t loss_ev) {
        const StageGeom &g = st[j];
        Worker &wr = wk[w];
        Flags *fl = flags_dev.as<Flags>();
        if (j == S - 1 && (launch_mask & 1)) {
            const int nt = std::max(32, round_up(B, 32));
            const size_t lsm = sizeof(double) * nt + sizeof(float) * B * g.dout;
            CDP_REQUIRE(lsm <= 220 * 1024, "loss kernel: batch x classes too large for shared memory");
            if (lsm > 48 * 1024)
                CDP_CUDA(cudaFuncSetAttribute(loss_kernel<K>, cudaFuncAttributeMaxDynamicSharedMemorySize, int(lsm)));
            launch_pdl(loss_kernel<K>, dim3(1), dim3(nt), lsm, s, (const float *)wr.z.as<float>(), B,
                       g.dout, loss_kind, perm_w, (const int *)data_lab.as<int>(), (const float *)data_tgt.as<float>(),
                       wr.dz[j].view(), wr.loss, &fl->loss);
            ++kernels_per_step;
        }
        if (loss_ev) CDP_CUDA(cudaEventRecord(loss_ev, s));
        if (j > 0 && (launch_mask & 2)) {
            Operand A[3], Bo[3];
            const int nseg = segments<K>(wc[vslot][j], false, g.din, g.dout, wr.dz[j], false, B, g.dout, A, Bo);
            typename EpiDgrad<K>::Params ep{rec[j][rin].view(), wr.dz[j - 1].view()};
            gemm<K, false, false, EpiDgrad<K>>(bn_rows(B), A, Bo, nseg, g.din, B, g.dout, wr, ep, s);
        }
    }

    // B task, hop half: [W; b] gradient ([h, 1]^T . dZ, M = din + 1) fused with
    // the ring hop / update.
    template <int K>
    void bwd_hop(int w, int j, int rin, int hop, int cur_slot, cudaStream_t s) {
        const StageGeom &g = st[j];
        Worker &wr = wk[w];
        Flags *fl = flags_dev.as<Flags>();
        Operand A[3], Bo[3];
        const int nseg = segments<K>(rec[j][rin], true, g.din + 1, B, wr.dz[j], true, g.dout, B, A, Bo);
        HopParams hp{};
        hp.mode = hop;
        hp.stage = j + 1;
        hp.base = g.base;
        hp.din = g.din;
        hp.dout = g.dout;
        hp.s_in = rank >= 0 ? prev_partial : partial;
        hp.s_out = partial;
        hp.theta_cur = theta[cur_slot];
        hp.theta_new = theta[cur_slot ^ 1];
        if (rank >= 0) {
            hp.sync.enabled = 1;
            hp.sync.n_readers = world - 1;
            hp.sync.step = &ctrl_dev.as<Control>()->step;
            hp.sync.own = ring;
            hp.sync.prev = prev_ring;
            hp.sync.cta_counter = cta_counters.as<unsigned>();
        }
        hp.vel = vel.as<float>();
        hp.lr = &ctrl_dev.as<Control>()->lr;
        hp.momentum = momentum;
        hp.wd = wd;
        hp.n_mb = float(rank >= 0 ? world : W);
        hp.wc_new = wc[cur_slot ^ 1][j].view();
        hp.grad_flags = &fl->grad;
        hp.upd_flags = &fl->upd;
        if (launch_mask & 4)
            gemm<K, true, true, EpiWgrad<K>>(bn_mn(g.dout), A, Bo, nseg, g.din + 1, g.dout, B, wr, hp, s);
    }

    // Both halves on one stream (operator-level timing helper).
    template <int K>
    void backward(int w, int j, int vslot, int rin, int hop, int cur_slot, cudaStream_t s, const int *perm_w) {
        bwd_compute<K>(w, j, vslot, rin, s, perm_w, nullptr);
        bwd_hop<K>(w, j, rin, hop, cur_slot, s);
    }

    // theta delivery on reader ranks (see pull_stage_kernel)
    template <int K>
    void pull(int j, int vslot, int fresh, cudaStream_t s) {
        CDP_REQUIRE(rank >= 0 && upd_ring && upd_theta[vslot], "pull op outside a connected multi-GPU trainer");
        const StageGeom &g = st[j];
        const int64_t n = int64_t(g.din) * g.dout + g.dout;
        const int blocks = int(std::min<int64_t>(148, (n + 1023) / 1024));
        launch_pdl(pull_stage_kernel<K>, dim3(blocks), dim3(256), 0, s, (const float *)(upd_theta[vslot] + g.base),
                   theta[vslot] + g.base, g.din, g.dout, wc[vslot][j].view(), upd_ring, ring, j + 1, fresh,
                   (const int *)&ctrl_dev.as<Control>()->step, cta_counters.as<unsigned>() + kMaxStages);
        ++kernels_per_step;
    }

    // ---------------------------------------------------------------- capture
    // Capture one training step.  Per worker two streams: the compute chain
    // (pull, F, loss, dgrad) and the hop stream (wgrad + fused hop / update),
    // so each layer's gradient hop overlaps the data-gradient chain below it.
    // Edges: hop(l) <- dZ_l ready; hop(l) <- dgrad(l) when the read was stale
    // (the update overwrites exactly that slot); ring B(i-1,l) -> B(i,l) on the
    // hop streams; slot reuse B -> producer F waits for both halves.
    template <int K>
    void record_step(int p) {
        kernels_per_step = 0;
        CDP_CUDA(cudaEventRecord(fork_ev, main));
        for (auto &w : wk) {
            CDP_CUDA(cudaStreamWaitEvent(w.stream, fork_ev, 0));
            CDP_CUDA(cudaStreamWaitEvent(w.hstream, fork_ev, 0));
        }
        std::vector<std::vector<int>> into(ops.size());
        for (auto &d : deps) into[d.second].push_back(d.first);
        std::vector<std::vector<cudaEvent_t>> dz_ready(W, std::vector<cudaEvent_t>(S, nullptr));
        uint64_t *tb = trace_buf.as<uint64_t>();
        auto stamp = [&](cudaStream_t st, int o, int k) {
            if (trace) {
                stamp_kernel<<<1, 1, 0, st>>>(tb + 4 * o + k);
                CDP_CUDA(cudaGetLastError());
            }
        };
        for (size_t o = 0; o < ops.size(); ++o) {
            const auto &op = ops[o];
            const int w = rank >= 0 ? 0 : op[OP_WORKER] - 1, j = op[OP_STAGE] - 1;
            cudaStream_t s = wk[w].stream, hs = wk[w].hstream;
            const int vslot = op[OP_FRESH] ? p : (p ^ 1);
            const int *perm_w = perm_dev.as<int>() + size_t(w) * B;
            if (op[OP_KIND] != 1) {
                for (int d : into[o]) {  // producer of a reused record slot: both halves of the releasing B
                    CDP_CUDA(cudaStreamWaitEvent(s, op_events[d], 0));
                    if (ops[d][OP_KIND] == 1) CDP_CUDA(cudaStreamWaitEvent(s, hop_events[d], 0));
                }
                stamp(s, int(o), 0);
                if (op[OP_KIND] == 2)
                    pull<K>(j, vslot, op[OP_FRESH], s);
                else
                    forward<K>(w, j, vslot, op[OP_REC_IN], op[OP_REC_OUT], s, perm_w);
                stamp(s, int(o), 1);
                CDP_CUDA(cudaEventRecord(op_events[o], s));
                continue;
            }
            stamp(s, int(o), 0);
            bwd_compute<K>(w, j, vslot, op[OP_REC_IN], s, perm_w, j == S - 1 ? loss_events[o] : nullptr);
            stamp(s, int(o), 1);
            CDP_CUDA(cudaEventRecord(op_events[o], s));
            if (j == S - 1) dz_ready[w][j] = loss_events[o];
            if (j > 0) dz_ready[w][j - 1] = op_events[o];
            CDP_REQUIRE(dz_ready[w][j] != nullptr, "plan runs a backward before the one producing its dZ");
            CDP_CUDA(cudaStreamWaitEvent(hs, dz_ready[w][j], 0));
            if (!op[OP_FRESH]) CDP_CUDA(cudaStreamWaitEvent(hs, op_events[o], 0));
            for (int d : into[o]) CDP_CUDA(cudaStreamWaitEvent(hs, ops[d][OP_KIND] == 1 ? hop_events[d] : op_events[d], 0));
            stamp(hs, int(o), 2);
            bwd_hop<K>(w, j, op[OP_REC_IN], op[OP_HOP], p, hs);
            stamp(hs, int(o), 3);
            CDP_CUDA(cudaEventRecord(hop_events[o], hs));
        }
        for (int w = 0; w < W; ++w) {
            CDP_CUDA(cudaEventRecord(join_ev[2 * w], wk[w].stream));
            CDP_CUDA(cudaStreamWaitEvent(main, join_ev[2 * w], 0));
            CDP_CUDA(cudaEventRecord(join_ev[2 * w + 1], wk[w].hstream));
            CDP_CUDA(cudaStreamWaitEvent(main, join_ev[2 * w + 1], 0));
        }
        finish_step();
    }

    void finish_step();

    void capture() {
        for (auto &e : exec)
            if (e) {
                CDP_CUDA(cudaGraphExecDestroy(e));
                e = nullptr;
            }
        for (auto *v : {&op_events, &hop_events, &loss_events, &join_ev}) {
            for (auto e : *v) cudaEventDestroy(e);
            v->clear();
        }
        if (fork_ev) {
            cudaEventDestroy(fork_ev);
            fork_ev = nullptr;
        }
        if (trace && !trace_buf.p) trace_buf = DevBuf(ops.size() * 4 * 8);
        for (auto *v : {&op_events, &hop_events, &loss_events}) {
            v->resize(ops.size());
            for (auto &e : *v) CDP_CUDA(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
        }
        join_ev.resize(2 * W);
        for (auto &e : join_ev) CDP_CUDA(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
        CDP_CUDA(cudaEventCreateWithFlags(&fork_ev, cudaEventDisableTiming));
        for (int p = 0; p < 2; ++p) {
            cudaGraph_t g;
            CDP_CUDA(cudaStreamBeginCapture(main, cudaStreamCaptureModeThreadLocal));
            try {
                if (kind == 0)
                    record_step<0>(p);
                else
                    record_step<1>(p);
            } catch (...) {
                // join the forked worker streams so the capture can be closed cleanly
                for (int w = 0; w < W; ++w) {
                    cudaEventRecord(join_ev[2 * w], wk[w].stream);
                    cudaStreamWaitEvent(main, join_ev[2 * w], 0);
                    cudaEventRecord(join_ev[2 * w + 1], wk[w].hstream);
                    cudaStreamWaitEvent(main, join_ev[2 * w + 1], 0);
                }
                if (cudaStreamEndCapture(main, &g) == cudaSuccess && g) cudaGraphDestroy(g);
                cudaGetLastError();
                throw;
            }
            CDP_CUDA(cudaStreamEndCapture(main, &g));
            CDP_CUDA(cudaGraphInstantiate(&exec[p], g, 0));
            CDP_CUDA(cudaGraphDestroy(g));
        }
    }

    // DP all-reduce baseline: apply the update of the step just run from the
    // (collective-summed) partial buffer, every layer, on the trainer stream.
    void apply_update() {
        CDP_REQUIRE(t >= 2, "no step has run");
        const int p = (t - 1) & 1;
        Flags *fl = flags_dev.as<Flags>();
        for (int j = 0; j < S; ++j) {
            const StageGeom &g = st[j];
            HopParams hp{};
            hp.mode = 3;
            hp.stage = j + 1;
            hp.base = g.base;
            hp.din = g.din;
            hp.dout = g.dout;
            hp.s_in = partial;
            hp.theta_cur = theta[p];
            hp.theta_new = theta[p ^ 1];
            hp.vel = vel.as<float>();
            hp.lr = &ctrl_dev.as<Control>()->lr;
            hp.momentum = momentum;
            hp.wd = wd;
            hp.n_mb = float(rank >= 0 ? world : W);
            hp.wc_new = wc[p ^ 1][j].view();
            hp.upd_flags = &fl->upd;
            const int64_t n = int64_t(g.din + 1) * g.dout;
            const int blocks = int(std::min<int64_t>(4 * 148, (n + 255) / 256));
            if (kind == 0)
                launch_pdl(update_from_sum_kernel<0>, dim3(blocks), dim3(256), 0, main, hp);
            else
                launch_pdl(update_from_sum_kernel<1>, dim3(blocks), dim3(256), 0, main, hp);
        }
    }

    // ---------------------------------------------------------------- params
    void pack_all(int slot) {
        for (int j = 0; j < S; ++j) {
            const float *w = theta[slot] + st[j].base;
            if (kind == 0)
                pack_w_kernel<0><<<148, 256, 0, main>>>(w, st[j].din, st[j].dout, wc[slot][j].view());
            else
                pack_w_kernel<1><<<148, 256, 0, main>>>(w, st[j].din, st[j].dout, wc[slot][j].view());
            CDP_CUDA(cudaGetLastError());
        }
    }

    void set_params(int which, const float *host) {
        // which: 0 = current (version t), 1 = previous (version t-1), -1 both
        for (int v = 0; v < 2; ++v) {
            if (which >= 0 && v != which) continue;
            const int slot = v == 0 ? (t & 1) : ((t & 1) ^ 1);
            CDP_CUDA(cudaMemcpyAsync(theta[slot], host, size_t(P) * 4, cudaMemcpyHostToDevice, main));
            pack_all(slot);
        }
        CDP_CUDA(cudaStreamSynchronize(main));
    }

    void get_params(int which, float *host) {
        CDP_CUDA(cudaStreamSynchronize(main));
        const int slot = which == 0 ? (t & 1) : ((t & 1) ^ 1);
        CDP_CUDA(cudaMemcpy(host, theta[slot], size_t(P) * 4, cudaMemcpyDeviceToHost));
    }

    void set_velocity(const float *host) {
        CDP_REQUIRE(vel.p != nullptr, "trainer has no momentum buffer");
        CDP_CUDA(cudaMemcpy(vel.p, host, size_t(P) * 4, cudaMemcpyHostToDevice));
    }
    void get_velocity(float *host) {
        CDP_REQUIRE(vel.p != nullptr, "trainer has no momentum buffer");
        CDP_CUDA(cudaStreamSynchronize(main));
        CDP_CUDA(cudaMemcpy(host, vel.p, size_t(P) * 4, cudaMemcpyDeviceToHost));
    }

    // One training step.  perm: W*B dataset row indices (micro-batch i = rows
    // [(i-1)B, iB)).  Asynchronous; results land in the history ring.
    void step(const int *perm, float lr) {
        const int k = stage_next;
        stage_next = (stage_next + 1) % RING;
        CDP_CUDA(cudaEventSynchronize(stage_ev[k]));  // the copy that last read this block has run
        uint8_t *blk = stage_host + size_t(k) * stage_bytes;
        Control *c = reinterpret_cast<Control *>(blk);
        c->lr = lr;
        c->step = t;
        std::memcpy(blk + sizeof(Control), perm, size_t(W) * B * 4);
        CDP_CUDA(cudaMemcpyAsync(ctrl_dev.p, blk, sizeof(Control), cudaMemcpyHostToDevice, main));
        CDP_CUDA(cudaMemcpyAsync(perm_dev.p, blk + sizeof(Control), size_t(W) * B * 4, cudaMemcpyHostToDevice, main));
        CDP_CUDA(cudaEventRecord(stage_ev[k], main));
        CDP_CUDA(cudaGraphLaunch(exec[t & 1], main));
        ++t;
    }

    // Launch one plan op's sub-kernels (mask) `iters` times, outside any graph, on
    // the main stream; returns the mean duration per iteration (CUDA events).
    // Destructive for the trainer state (re-applies hops / updates): bench only.
    float time_op(int o, int mask, int iters) {
        CDP_REQUIRE(o >= 0 && o < int(ops.size()), "op index out of range");
        const auto &op = ops[o];
        const int w = op[OP_WORKER] - 1, j = op[OP_STAGE] - 1;
        const int p = t & 1, vslot = op[OP_FRESH] ? p : (p ^ 1);
        const int *perm_w = perm_dev.as<int>() + size_t(w) * B;
        cudaEvent_t e0, e1;
        CDP_CUDA(cudaEventCreate(&e0));
        CDP_CUDA(cudaEventCreate(&e1));
        launch_mask = mask;
        auto run = [&] {
            if (op[OP_KIND] == 0) {
                if (kind == 0) forward<0>(w, j, vslot, op[OP_REC_IN], op[OP_REC_OUT], main, perm_w);
                else forward<1>(w, j, vslot, op[OP_REC_IN], op[OP_REC_OUT], main, perm_w);
            } else {
                if (kind == 0) backward<0>(w, j, vslot, op[OP_REC_IN], op[OP_HOP], p, main, perm_w);
                else backward<1>(w, j, vslot, op[OP_REC_IN], op[OP_HOP], p, main, perm_w);
            }
        };
        const int saved = kernels_per_step;
        const bool warm = iters > 0;  // iters < 0: cold (no warm-up launch), |iters| launches
        iters = iters > 0 ? iters : -iters;
        if (warm) run();
        CDP_CUDA(cudaEventRecord(e0, main));
        for (int i = 0; i < iters; ++i) run();
        CDP_CUDA(cudaEventRecord(e1, main));
        CDP_CUDA(cudaEventSynchronize(e1));
        launch_mask = 7;
        kernels_per_step = saved;
        float ms = 0.f;
        CDP_CUDA(cudaEventElapsedTime(&ms, e0, e1));
        cudaEventDestroy(e0);
        cudaEventDestroy(e1);
        return ms / iters;
    }

    void mark(int k) {
        while (int(marks.size()) <= k) {
            cudaEvent_t e;
            CDP_CUDA(cudaEventCreate(&e));
            marks.push_back(e);
        }
        CDP_CUDA(cudaEventRecord(marks[k], main));
    }

    void flush_l2() {
        if (!flush_buf.p) flush_buf = DevBuf(size_t(256) << 20);
        CDP_CUDA(cudaMemsetAsync(flush_buf.p, t & 0xff, flush_buf.bytes, main));
    }

    // Host-batch step (end-to-end path): the step's inputs come from host memory.
    void step_host_batch(const float *x, const int *labels, const float *targets, float lr) {
        const size_t rows = size_t(W) * B;
        CDP_CUDA(cudaMemcpyAsync(data_x.p, x, rows * st[0].din * 4, cudaMemcpyHostToDevice, main));
        if (loss_kind == 1)
            CDP_CUDA(cudaMemcpyAsync(data_lab.p, labels, rows * 4, cudaMemcpyHostToDevice, main));
        else
            CDP_CUDA(cudaMemcpyAsync(data_tgt.p, targets, rows * st[S - 1].dout * 4, cudaMemcpyHostToDevice, main));
        std::vector<int> ident(rows);
        for (size_t r = 0; r < rows; ++r) ident[r] = int(r);
        step(ident.data(), lr);
    }
};

__global__ void finish_step_kernel(const double *losses, int W, Flags *flags, double *hist_loss, Flags *hist_flags,
                                   int *hist_count, int cap) {
    double acc = 0.0;
    for (int w = 0; w < W; ++w) acc += losses[w];  // ascending micro-batch (ref engine.py:96)
    const int c = *hist_count;
    hist_loss[c % cap] = acc / W;  // ring of the last `cap` steps
    hist_flags[c % cap] = *flags;
    *hist_count = c + 1;
    *flags = Flags{0, 0, 0, 0};
}

void MlpTrainer::finish_step() {
    finish_step_kernel<<<1, 1, 0, main>>>(loss_all.as<double>(), W, flags_dev.as<Flags>(), hist_loss.as<double>(),
                                          hist_flags.as<Flags>(), hist_count.as<int>(), hist_cap);
    CDP_CUDA(cudaGetLastError());
    ++kernels_per_step;
}

}  // namespace cdp

using namespace cdp;

struct cdp_trainer {
    std::unique_ptr<MlpTrainer> impl;
};

static std::unique_ptr<MlpTrainer> create_impl(int n_dims, const int64_t *dims, int micro_batch, int n_workers,
                                               int loss_kind, int dtype, float momentum, float weight_decay, int n_ops,
                                               const int32_t *ops, int n_deps, const int32_t *deps,
                                               const int32_t *slots_per_stage, int n_samples, const float *x,
                                               const int32_t *labels, const float *targets, int rank, int world) {
    CDP_REQUIRE(dtype == CDP_DTYPE_FP32 || dtype == CDP_DTYPE_BF16, "dtype must be CDP_DTYPE_FP32 or CDP_DTYPE_BF16");
    CDP_REQUIRE(loss_kind == 0 || loss_kind == 1, "loss_kind must be 0 (mse) or 1 (xent)");
    CDP_REQUIRE(n_workers >= 1, "n_workers must be >= 1");
    CDP_REQUIRE(n_dims - 1 <= kMaxStages, "too many stages");
    auto tr = std::make_unique<MlpTrainer>();
    tr->kind = dtype == CDP_DTYPE_BF16 ? 0 : 1;
    tr->rank = rank;
    tr->world = world;
    tr->W = rank >= 0 ? 1 : n_workers;
    tr->B = micro_batch;
    tr->loss_kind = loss_kind;
    tr->momentum = momentum;
    tr->wd = weight_decay;
    tr->slots.assign(n_dims, 1);
    for (int j = 1; j < n_dims; ++j) tr->slots[j] = slots_per_stage[j];
    for (int o = 0; o < n_ops; ++o) {
        std::array<int, OP_FIELDS> a;
        for (int f = 0; f < OP_FIELDS; ++f) a[f] = ops[o * OP_FIELDS + f];
        CDP_REQUIRE(a[OP_KIND] >= 0 && a[OP_KIND] <= 2, "op kind must be 0 (F), 1 (B) or 2 (pull)");
        CDP_REQUIRE(a[OP_WORKER] >= 1 && a[OP_WORKER] <= n_workers, "op worker out of range");
        CDP_REQUIRE(rank < 0 || a[OP_WORKER] == rank + 1, "a rank's plan may only hold its own worker's ops");
        CDP_REQUIRE(a[OP_KIND] != 2 || rank >= 0, "pull ops need a multi-GPU trainer");
        CDP_REQUIRE(a[OP_STAGE] >= 1 && a[OP_STAGE] < n_dims, "op stage out of range");
        tr->ops.push_back(a);
    }
    for (int d = 0; d < n_deps; ++d) {
        CDP_REQUIRE(deps[2 * d] < deps[2 * d + 1], "plan edges must point forward in op order");
        tr->deps.emplace_back(deps[2 * d], deps[2 * d + 1]);
    }
    tr->setup(dims, n_dims);
    for (auto &op : tr->ops) {
        if (op[OP_KIND] == 2) continue;
        CDP_REQUIRE(op[OP_REC_IN] < tr->slots[op[OP_STAGE]], "record slot out of range");
        if (op[OP_KIND] == 0 && op[OP_STAGE] < tr->S)
            CDP_REQUIRE(op[OP_REC_OUT] < tr->slots[op[OP_STAGE] + 1], "record slot out of range");
    }
    tr->upload_data(n_samples, x, labels, targets);
    return tr;
}

extern "C" int cdp_trainer_create(int n_dims, const int64_t *dims, int micro_batch, int n_workers, int loss_kind,
                                  int dtype, float momentum, float weight_decay, int n_ops, const int32_t *ops,
                                  int n_deps, const int32_t *deps, const int32_t *slots_per_stage, int n_samples,
                                  const float *x, const int32_t *labels, const float *targets, cdp_trainer **out) {
    return guarded([&] {
        auto tr = create_impl(n_dims, dims, micro_batch, n_workers, loss_kind, dtype, momentum, weight_decay, n_ops,
                              ops, n_deps, deps, slots_per_stage, n_samples, x, labels, targets, -1, 1);
        tr->capture();
        *out = new cdp_trainer{std::move(tr)};
    });
}

extern "C" int cdp_trainer_create_rank(int n_dims, const int64_t *dims, int micro_batch, int world, int rank,
                                       int loss_kind, int dtype, float momentum, float weight_decay, int n_ops,
                                       const int32_t *ops, int n_samples, const float *x, const int32_t *labels,
                                       const float *targets, cdp_trainer **out) {
    return guarded([&] {
        CDP_REQUIRE(world >= 1 && rank >= 0 && rank < world, "bad rank / world");
        std::vector<int32_t> slots(n_dims, 1);
        auto tr = create_impl(n_dims, dims, micro_batch, world, loss_kind, dtype, momentum, weight_decay, n_ops, ops,
                              0, nullptr, slots.data(), n_samples, x, labels, targets, rank, world);
        *out = new cdp_trainer{std::move(tr)};
    });
}

extern "C" int cdp_trainer_region(cdp_trainer *tr, void **base, size_t *bytes) {
    return guarded([&] {
        *base = tr->impl->region.p;
        *bytes = tr->impl->region.bytes;
    });
}

extern "C" int cdp_trainer_ipc_handle(cdp_trainer *tr, void *handle64) {
    return guarded([&] {
        cudaIpcMemHandle_t h;
        CDP_CUDA(cudaIpcGetMemHandle(&h, tr->impl->region.p));
        std::memcpy(handle64, &h, sizeof(h));
    });
}

extern "C" int cdp_ipc_open(const void *handle64, void **ptr) {
    return guarded([&] {
        cudaIpcMemHandle_t h;
        std::memcpy(&h, handle64, sizeof(h));
        CDP_CUDA(cudaIpcOpenMemHandle(ptr, h, cudaIpcMemLazyEnablePeerAccess));
    });
}

extern "C" int cdp_ipc_close(void *ptr) {
    return guarded([&] { CDP_CUDA(cudaIpcCloseMemHandle(ptr)); });
}

// regions[r] = base of rank r's shared region, valid in this process (own
// region for r == rank; IPC-mapped or same-process pointers for peers).
extern "C" int cdp_trainer_connect(cdp_trainer *tr, void *const *regions) {
    return guarded([&] {
        auto &m = *tr->impl;
        CDP_REQUIRE(m.rank >= 0, "connect is for multi-GPU (per-rank) trainers");
        auto at = [&](int r) { return static_cast<uint8_t *>(regions[r]); };
        const size_t off = m.region_theta_off;
        if (m.rank > 0) {
            m.prev_ring = reinterpret_cast<RingFlags *>(at(m.rank - 1));
            m.prev_partial = reinterpret_cast<float *>(at(m.rank - 1) + off) + 2 * m.Pp;
        }
        const int u = m.world - 1;
        m.upd_ring = reinterpret_cast<RingFlags *>(at(u));
        m.upd_theta[0] = reinterpret_cast<float *>(at(u) + off);
        m.upd_theta[1] = m.upd_theta[0] + m.Pp;
        m.capture();
    });
}

// Non-zero when a cross-GPU spin-wait timed out (protocol failure).
extern "C" int cdp_trainer_ring_error(cdp_trainer *tr, int *err) {
    return guarded([&] {
        CDP_CUDA(cudaStreamSynchronize(tr->impl->main));
        uint32_t e = 0;
        CDP_CUDA(cudaMemcpy(&e, &tr->impl->ring->err, 4, cudaMemcpyDeviceToHost));
        *err = int(e);
    });
}

extern "C" void cdp_trainer_destroy(cdp_trainer *tr) {
    if (tr) {
        cudaDeviceSynchronize();
        delete tr;
    }
}

extern "C" int cdp_trainer_set_params(cdp_trainer *tr, int which, const float *theta) {
    return guarded([&] { tr->impl->set_params(which, theta); });
}

extern "C" int cdp_trainer_get_params(cdp_trainer *tr, int which, float *theta) {
    return guarded([&] { tr->impl->get_params(which, theta); });
}

extern "C" int cdp_trainer_set_velocity(cdp_trainer *tr, const float *v) {
    return guarded([&] { tr->impl->set_velocity(v); });
}

extern "C" int cdp_trainer_get_velocity(cdp_trainer *tr, float *v) {
    return guarded([&] { tr->impl->get_velocity(v); });
}

extern "C" int cdp_trainer_step(cdp_trainer *tr, const int32_t *perm, float lr) {
    return guarded([&] { tr->impl->step(perm, lr); });
}

extern "C" int cdp_trainer_step_host_batch(cdp_trainer *tr, const float *x, const int32_t *labels,
                                           const float *targets, float lr) {
    return guarded([&] { tr->impl->step_host_batch(x, labels, targets, lr); });
}

extern "C" int cdp_trainer_sync(cdp_trainer *tr) {
    return guarded([&] { CDP_CUDA(cudaStreamSynchronize(tr->impl->main)); });
}

extern "C" int cdp_trainer_history(cdp_trainer *tr, int max, double *losses, uint32_t *flags, int *count) {
    return guarded([&] {
        auto &m = *tr->impl;
        CDP_CUDA(cudaStreamSynchronize(m.main));
        int c = 0;
        CDP_CUDA(cudaMemcpy(&c, m.hist_count.p, 4, cudaMemcpyDeviceToHost));
        *count = c;
        // oldest retained step first: steps [c - n, c) live at ring index k % cap
        const int n = std::min({c, max, m.hist_cap});
        if (n > 0) {
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
        }
    });
}

extern "C" int cdp_trainer_stats(cdp_trainer *tr, int64_t *out, int n_out) {
    // [0] activation-record bytes, [1] parameter-state bytes, [2] kernels per step,
    // [3] step (next), [4] stream count, [5] ops per step
    return guarded([&] {
        auto &m = *tr->impl;
        int64_t act = 0;
        for (auto &stage : m.rec)
            for (auto &r : stage) act += int64_t(r.hi.bytes + r.lo.bytes);
        int64_t par = int64_t(m.P) * 4 * 3 + int64_t(m.vel.bytes);
        for (int v = 0; v < 2; ++v)
            for (auto &c : m.wc[v]) par += int64_t(c.hi.bytes + c.lo.bytes);
        int64_t vals[6] = {act, par, m.kernels_per_step, m.t, int64_t(m.W), int64_t(m.ops.size())};
        for (int i = 0; i < n_out && i < 6; ++i) out[i] = vals[i];
    });
}

extern "C" int cdp_trainer_get_grad(cdp_trainer *tr, float *grad) {
    return guarded([&] {
        auto &m = *tr->impl;
        CDP_CUDA(cudaStreamSynchronize(m.main));
        CDP_CUDA(cudaMemcpy(grad, m.partial, size_t(m.P) * 4, cudaMemcpyDeviceToHost));
    });
}

extern "C" int cdp_trainer_stream(cdp_trainer *tr, void **stream) {
    return guarded([&] { *stream = tr->impl->main; });
}

// ---------------------------------------------------------------------------
// Operator level (ref training/_kernels.pyx:25-132, backend protocol
// training/backend.py:13-30): value + flat gradient of one micro-batch, host
// fp64 in / out.  Runs the same fused layer kernels as the trainer through a
// cached single-worker plan whose B tasks write the raw gradient (hop mode 4).
namespace {
std::mutex g_vg_mu;
std::map<std::vector<int64_t>, std::unique_ptr<MlpTrainer>> g_vg_cache;

MlpTrainer &value_grad_trainer(int n_dims, const int64_t *dims, int batch, int loss_kind, int dtype) {
    std::vector<int64_t> key(dims, dims + n_dims);
    key.push_back(batch);
    key.push_back(loss_kind);
    key.push_back(dtype);
    auto it = g_vg_cache.find(key);
    if (it != g_vg_cache.end()) return *it->second;
    auto tr = std::make_unique<MlpTrainer>();
    tr->kind = dtype == CDP_DTYPE_BF16 ? 0 : 1;
    tr->W = 1;
    tr->B = batch;
    tr->loss_kind = loss_kind;
    const int S = n_dims - 1;
    tr->slots.assign(n_dims, 1);
    for (int j = 1; j <= S; ++j) tr->ops.push_back({0, 1, j, 1, 0, 0, 0, 0});
    for (int j = S; j >= 1; --j) tr->ops.push_back({1, 1, j, 1, 0, 0, HOP_GRAD, 0});
    tr->setup(dims, n_dims);
    tr->upload_data(batch, nullptr, nullptr, nullptr);
    tr->capture();
    auto &ref = *tr;
    g_vg_cache.emplace(std::move(key), std::move(tr));
    return ref;
}
}  // namespace

extern "C" int cdp_mlp_value_grad(int n_dims, const int64_t *dims, const double *theta, int batch, const double *x,
                                  const double *y, const int64_t *labels, int loss_kind, int dtype, double *loss_out,
                                  double *grad_out) {
    return guarded([&] {
        CDP_REQUIRE(n_dims >= 2, "dims needs at least input and output widths");
        CDP_REQUIRE(loss_kind == 0 || loss_kind == 1, "loss_kind must be 0 (mse) or 1 (xent)");
        CDP_REQUIRE(dtype == CDP_DTYPE_FP32 || dtype == CDP_DTYPE_BF16, "bad dtype");
        CDP_REQUIRE(loss_kind == 0 ? y != nullptr : labels != nullptr, "missing targets");
        std::lock_guard<std::mutex> lk(g_vg_mu);
        MlpTrainer &tr = value_grad_trainer(n_dims, dims, batch, loss_kind, dtype);
        std::vector<float> th(tr.P);
        for (int64_t i = 0; i < tr.P; ++i) th[i] = float(theta[i]);
        tr.set_params(-1, th.data());
        const int din = int(dims[0]), dout = int(dims[n_dims - 1]);
        std::vector<float> xf(size_t(batch) * din), yf;
        std::vector<int> lab;
        for (size_t i = 0; i < xf.size(); ++i) xf[i] = float(x[i]);
        if (loss_kind == 0) {
            yf.resize(size_t(batch) * dout);
            for (size_t i = 0; i < yf.size(); ++i) yf[i] = float(y[i]);
        } else {
            lab.resize(batch);
            for (int i = 0; i < batch; ++i) {
                CDP_REQUIRE(labels[i] >= 0 && labels[i] < dout, "label out of range");
                lab[i] = int(labels[i]);
            }
        }
        tr.step_host_batch(xf.data(), lab.data(), yf.data(), 0.f);
        CDP_CUDA(cudaStreamSynchronize(tr.main));
        int c = 0;
        CDP_CUDA(cudaMemcpy(&c, tr.hist_count.p, 4, cudaMemcpyDeviceToHost));
        CDP_CUDA(cudaMemcpy(loss_out, tr.hist_loss.as<double>() + (c - 1) % tr.hist_cap, 8, cudaMemcpyDeviceToHost));
        std::vector<float> g(tr.P);
        CDP_CUDA(cudaMemcpy(g.data(), tr.partial, size_t(tr.P) * 4, cudaMemcpyDeviceToHost));
        for (int64_t i = 0; i < tr.P; ++i) grad_out[i] = double(g[i]);
    });
}

extern "C" int cdp_trainer_last(cdp_trainer *tr, double *loss, uint32_t *flags) {
    return guarded([&] {
        auto &m = *tr->impl;
        CDP_CUDA(cudaStreamSynchronize(m.main));
        const int c = m.t - 1;  // steps launched (and now finished)
        CDP_REQUIRE(c >= 1, "no step has run");
        const int k = (c - 1) % m.hist_cap;
        Flags f;
        CDP_CUDA(cudaMemcpy(loss, m.hist_loss.as<double>() + k, 8, cudaMemcpyDeviceToHost));
        CDP_CUDA(cudaMemcpy(&f, m.hist_flags.as<Flags>() + k, sizeof(Flags), cudaMemcpyDeviceToHost));
        flags[0] = f.grad;
        flags[1] = f.loss;
        flags[2] = f.upd;
    });
}

extern "C" int cdp_trainer_time_op(cdp_trainer *tr, int op, int mask, int iters, float *ms) {
    return guarded([&] { *ms = tr->impl->time_op(op, mask, iters); });
}

extern "C" int cdp_trainer_mark(cdp_trainer *tr, int k) {
    return guarded([&] { tr->impl->mark(k); });
}

extern "C" int cdp_trainer_elapsed(cdp_trainer *tr, int a, int b, float *ms) {
    return guarded([&] {
        auto &m = *tr->impl;
        CDP_REQUIRE(a >= 0 && b >= 0 && a < int(m.marks.size()) && b < int(m.marks.size()), "mark out of range");
        CDP_CUDA(cudaEventSynchronize(m.marks[b]));
        CDP_CUDA(cudaEventElapsedTime(ms, m.marks[a], m.marks[b]));
    });
}

extern "C" int cdp_trainer_flush_l2(cdp_trainer *tr) {
    return guarded([&] { tr->impl->flush_l2(); });
}

extern "C" int cdp_trainer_partial(cdp_trainer *tr, void **ptr, size_t *n_floats) {
    return guarded([&] {
        *ptr = tr->impl->partial;
        *n_floats = size_t(tr->impl->P);
    });
}

extern "C" int cdp_trainer_apply_update(cdp_trainer *tr) {
    return guarded([&] { tr->impl->apply_update(); });
}

extern "C" int cdp_trainer_set_trace(cdp_trainer *tr, int on) {
    return guarded([&] {
        auto &m = *tr->impl;
        CDP_CUDA(cudaStreamSynchronize(m.main));
        m.trace = on != 0;
        m.capture();
    });
}

extern "C" int cdp_trainer_trace(cdp_trainer *tr, uint64_t *out, int n_ops) {
    return guarded([&] {
        auto &m = *tr->impl;
        CDP_REQUIRE(m.trace_buf.p, "trace mode was never enabled");
        CDP_REQUIRE(n_ops == int(m.ops.size()), "n_ops must equal the plan's op count");
        CDP_CUDA(cudaStreamSynchronize(m.main));
        CDP_CUDA(cudaMemcpy(out, m.trace_buf.p, m.ops.size() * 4 * 8, cudaMemcpyDeviceToHost));
    });
}
