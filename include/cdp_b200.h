/*
 * cdp_b200.h — C ABI of libcdp_b200.so, the sm_100a implementation of the
 * Cyclic Data Parallelism training step (arXiv 2403.08837).
 *
 * Plain C types only (pointers, sizes, ints, floats); no torch types.  Every
 * entry point returns 0 on success and non-zero on failure, with the message
 * available from cdp_last_error() (thread-local).  The Python side
 * (paper_2403_08837_b200/_native.py) binds these with ctypes; INTEGRATION.md
 * shows the binding a maintainer of the reference would add.
 *
 * Reference interfaces replaced (all paths under /root/reference/pkg/src/cyclicdp):
 *   cdp_mlp_value_grad   <- training/_kernels.pyx:25-132 `mlp_value_grad`
 *                           (backend protocol training/backend.py:13-30,
 *                            called from training/models.py:84-88)
 *   cdp_quad_value_grad  <- training/_kernels.pyx:135-172 `quad_value_grad`
 *                           (called from training/models.py:148)
 *   cdp_trainer_*        <- training/engine.py:66-116 `_advance` and its
 *                           drivers step_dp / step_cdp / run_experiment
 *                           (engine.py:119-215): the whole training step,
 *                           device resident, one CUDA graph per step.
 *   cdp_resnet_* / cdp_vit_*  <- the same step for the named models, one worker per
 *                           process (rank): the comm.py:37-67 `schedule_cdp_ring_reduce`
 *                           hop and the engine.py:96-109 accumulate / update run inside
 *                           the weight-gradient GEMM epilogues over peer memory; the
 *                           comm.py:126-143 ZeRO-CDP STATE_TRANSFER runs as peer state
 *                           copies inside the step (cdp_resnet_create_rank zero_table).
 *                           There is no separate hop or shard-copy entry point: both are
 *                           fused into the step graph.
 */
#ifndef CDP_B200_H
#define CDP_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* ---- library ---------------------------------------------------------- */
const char *cdp_last_error(void);
int cdp_version(void);
/* Number of SMs of the current device (0 if no device). */
int cdp_device_sm_count(void);
/* Select the device of the calling thread for this library's CUDA runtime (the library links its own
 * runtime; the Python layer binds it to torch's current device, one process per GPU). */
int cdp_set_device(int device);
/* Synchronous device -> host copy (tests / diagnostics read internal buffers with it). */
int cdp_memcpy_d2h(void *dst, const void *src, size_t bytes);

/* Compute precision of the layer kernels. */
enum cdp_dtype {
    CDP_DTYPE_FP32 = 0, /* fp32 storage, 3xTF32 tcgen05 products (fp32-accurate) */
    CDP_DTYPE_BF16 = 1  /* bf16 operands, fp32 accumulate, fp32 master params   */
};

/* ---- operator level: the reference backend protocol ------------------- */
/* Loss and flat gradient of the stage-stacked tanh MLP on one micro-batch.
 * Host fp64 buffers in the reference layout (per stage W[din][dout] then
 * b[dout]); loss_kind 0 = MSE against y[batch][dims[n-1]], 1 = softmax
 * cross-entropy against labels[batch].  grad_out is fully overwritten. */
int cdp_mlp_value_grad(int n_dims, const int64_t *dims, const double *theta, int batch, const double *x,
                       const double *y, const int64_t *labels, int loss_kind, int dtype, double *loss_out,
                       double *grad_out);

/* 0.5*|A theta - t|^2 averaged over rows and batch; a is [m][p]. */
int cdp_quad_value_grad(int m, int p, const double *a, const double *theta, int batch, const double *targets,
                        double *loss_out, double *grad_out);

/* ---- step level: the device-resident CDP / DP trainer ---------------- */
/* Replaces ref training/engine.py:66-116 (_advance) for the stage MLP.  The
 * step plan comes from the reference-parity Timeline
 * (paper_2403_08837_b200/executor.py): ops[n_ops][8] =
 *   {kind 0=F/1=B, worker i (1-based), stage j (1-based), fresh (rule table),
 *    input-record slot, output-record slot, hop role, 0}
 * with hop role 0 first / 1 middle / 2 last (fused SGD update) / 3 only /
 * 4 gradient only; deps[n_deps][2] = cross-worker edges (before, after);
 * slots_per_stage[n_dims] = activation-record slots (index 0 unused).
 * Dataset (optional, n_samples rows): x fp32 [n][dims[0]], labels int32 [n]
 * (loss_kind 1) or targets fp32 [n][dims[n_dims-1]] (loss_kind 0). */
typedef struct cdp_trainer cdp_trainer;
int cdp_trainer_create(int n_dims, const int64_t *dims, int micro_batch, int n_workers, int loss_kind, int dtype,
                       float momentum, float weight_decay, int n_ops, const int32_t *ops, int n_deps,
                       const int32_t *deps, const int32_t *slots_per_stage, int n_samples, const float *x,
                       const int32_t *labels, const float *targets, cdp_trainer **out);
void cdp_trainer_destroy(cdp_trainer *tr);

/* ---- multi-GPU CDP: one process (rank) per GPU, worker i = rank + 1 ------ */
/* The rank's plan holds only its own worker's ops plus pull ops (kind 2:
 * fetch the version of stage j this worker is about to read from the
 * updater rank world-1).  The gradient hop of B(i,j) reads rank i-2's
 * partial sum from peer HBM (ref comm.py:37-67), the last rank fuses the
 * update.  Synchronisation is by step-numbered flags in each rank's shared
 * region (st.release.sys / ld.acquire.sys); spin-waits time out (~2 s) into
 * cdp_trainer_ring_error instead of hanging.  Sequence: create_rank ->
 * (ipc_handle, exchange, ipc_open peers) -> connect(regions) -> steps. */
int cdp_trainer_create_rank(int n_dims, const int64_t *dims, int micro_batch, int world, int rank, int loss_kind,
                            int dtype, float momentum, float weight_decay, int n_ops, const int32_t *ops,
                            int n_samples, const float *x, const int32_t *labels, const float *targets,
                            cdp_trainer **out);
/* Base / size of the rank's shared region (flags, both parameter slots, partial sum). */
int cdp_trainer_region(cdp_trainer *tr, void **base, size_t *bytes);
/* 64-byte cudaIpcMemHandle_t of the shared region. */
int cdp_trainer_ipc_handle(cdp_trainer *tr, void *handle64);
int cdp_ipc_open(const void *handle64, void **ptr);
int cdp_ipc_close(void *ptr);
/* regions[r] = rank r's region base, valid in this process; captures the step graphs. */
int cdp_trainer_connect(cdp_trainer *tr, void *const *regions);
int cdp_trainer_ring_error(cdp_trainer *tr, int *err);
/* DP all-reduce baseline (ref comm.py:70-90): plans whose B ops use hop role 4
 * leave each rank's own micro-batch gradient in the partial buffer; the host
 * all-reduces it (NCCL) on the trainer stream, then apply_update runs the SGD
 * update of the step just run on every replica. */
int cdp_trainer_partial(cdp_trainer *tr, void **ptr, size_t *n_floats);
int cdp_trainer_apply_update(cdp_trainer *tr);
/* which: 0 = current version (theta_t), 1 = previous (theta_{t-1}), -1 = both.
 * Flat fp32 host buffers in the reference layout. */
int cdp_trainer_set_params(cdp_trainer *tr, int which, const float *theta);
int cdp_trainer_get_params(cdp_trainer *tr, int which, float *theta);
int cdp_trainer_set_velocity(cdp_trainer *tr, const float *v);
int cdp_trainer_get_velocity(cdp_trainer *tr, float *v);
/* One training step (asynchronous): perm = n_workers*micro_batch dataset rows,
 * micro-batch i = perm[(i-1)B, iB) (ref training/models.py:173-181). */
int cdp_trainer_step(cdp_trainer *tr, const int32_t *perm, float lr);
/* One step whose inputs are host buffers (n_workers*micro_batch rows, copied
 * H2D inside the step): the end-to-end path. */
int cdp_trainer_step_host_batch(cdp_trainer *tr, const float *x, const int32_t *labels, const float *targets,
                                float lr);
int cdp_trainer_sync(cdp_trainer *tr);
/* Mean loss and non-finite flags {grad stage bits, loss, update stage bits}
 * of the retained steps, oldest first; *count = steps run so far. */
int cdp_trainer_history(cdp_trainer *tr, int max, double *losses, uint32_t *flags, int *count);
/* out[0..5] = activation-record bytes, parameter-state bytes, kernels per
 * step, next step index, worker streams, ops per step. */
int cdp_trainer_stats(cdp_trainer *tr, int64_t *out, int n_out);
/* The partial-sum buffer (gradient of the last step in gradient-only plans). */
int cdp_trainer_get_grad(cdp_trainer *tr, float *grad);
/* Mean loss and flags of the most recent step (synchronises the trainer stream). */
int cdp_trainer_last(cdp_trainer *tr, double *loss, uint32_t *flags);
/* Measurement helpers (bench.py): launch op `op`'s sub-kernels selected by
 * mask (1 gather/loss, 2 fwd/dgrad GEMM, 4 wgrad+hop GEMM) `iters` times
 * outside the graph and return the mean ms per iteration (destructive to the
 * trainer state); timing events on the trainer stream; L2 flush (256 MiB). */
int cdp_trainer_time_op(cdp_trainer *tr, int op, int mask, int iters, float *ms);
int cdp_trainer_mark(cdp_trainer *tr, int k);
int cdp_trainer_elapsed(cdp_trainer *tr, int a, int b, float *ms);
int cdp_trainer_flush_l2(cdp_trainer *tr);
/* Trace mode (re-captures the step graphs): %globaltimer stamps around every
 * op; cdp_trainer_trace returns [n_ops][4] u64 = compute start, compute end,
 * hop start, hop end (0 for ops without a hop half) of the last step. */
int cdp_trainer_set_trace(cdp_trainer *tr, int on);
int cdp_trainer_trace(cdp_trainer *tr, uint64_t *out, int n_ops);
/* The cudaStream_t the step graphs are launched on. */
int cdp_trainer_stream(cdp_trainer *tr, void **stream);

/* ---- ResNets (BASELINE configs[1..2,4]: ResNet-18 CIFAR, ResNet-50 ImageNet) */
/* One worker per process (rank of world; world = 1 = single GPU).  Replaces the
 * per-micro-batch value+grad + _advance accumulate/update of the reference
 * (training/engine.py:66-116) for a convolutional model.  Layers: stem
 * (stem_kind 0: 3x3/s1 conv, CIFAR; 1: 7x7/s2 conv + 3x3/s2 max pool,
 * ImageNet) + BN + ReLU, then per stage l depths[l] blocks (block_kind 0:
 * BasicBlock of width widths[l]; 1: Bottleneck of width widths[l], expansion
 * 4); the first block of stage l > 0 has stride 2 (on the 3x3 conv) and a 1x1
 * projection shortcut whenever the shape changes; global average pool,
 * classifier.  Parameter tensors (hop units) in torchvision order: conv
 * [R*S*Cin][Cout], BN [gamma(C) | beta(C)], fc [[W^T]; b] = [C+1][classes];
 * tensor_stage[i] (1-based) groups them into world stages, stage_fresh[s] =
 * this rank's rule row.  Dataset: x fp32 NHWC [n][height][width][in_channels],
 * labels int32. */
typedef struct cdp_resnet cdp_resnet;
int cdp_resnet_create_rank(int n_layers, const int32_t *widths, const int32_t *depths, int block_kind, int stem_kind,
                           int in_channels, int height, int width, int classes, int micro_batch, int world, int rank,
                           const int32_t *tensor_stage, const uint8_t *stage_fresh, int dtype, float momentum,
                           float weight_decay, int n_samples, const float *x, const int32_t *labels,
                           const int32_t *zero_table, int options, cdp_resnet **out);
/* options bit 0: DP all-reduce baseline (ref comm.py:70-90): the weight-gradient epilogues write this
 * rank's gradient into the flat buffer (cdp_resnet_partial); the caller sums it across ranks on the
 * trainer stream (cdp_resnet_stream, e.g. ncclAllReduce) and calls cdp_resnet_apply_update. */
int cdp_resnet_apply_update(cdp_resnet *tr);
/* ZeRO-DP baseline (ref comm.py:108-124: the owner of each stage broadcasts its states, the
 * gradients are reduced to the owner): the owner updates only its tensors [first, end), the
 * non-owners repack the compute copies of the tensors written into theta slot `which` (0 current,
 * 1 previous; cdp_resnet_buffer "theta") by the caller's broadcast. */
int cdp_resnet_apply_update_range(cdp_resnet *tr, int first_tensor, int end_tensor);
int cdp_resnet_pack_range(cdp_resnet *tr, int which, int first_tensor, int end_tensor);
int cdp_resnet_partial(cdp_resnet *tr, void **ptr, size_t *n);
int cdp_resnet_stream(cdp_resnet *tr, void **stream);
/* zero_table != NULL (world > 1): ZeRO-CDP state passing (ref comm.py:93-144), [world stages][2 (F, B)]
 * [world ranks][3] = (use-index base, predecessor rank, predecessor step offset) from zero.py; every
 * use of a parameter tensor copies the tensor's state (both theta slots + momentum) from its
 * predecessor's HBM.  The state lives in two stage frames per rank (ref schedule.py:449-458: a worker
 * holds only the stage it uses; stage s in frame (s - 1) & 1, frames reused once the successor copied
 * them); options bit 2 keeps full replicas instead.  cdp_resnet_zero_drain publishes the forward uses
 * of the next (unlaunched) step at the end of a run (call on every rank before synchronising). */
int cdp_resnet_zero_drain(cdp_resnet *tr);
/* ZeRO-CDP frames: this rank's frame contents in the full parameter layout (which 0: current version,
 * 1: previous) and its last finished use index per tensor (last_use[n_tensors]); the newest state of a
 * tensor is on the rank with the largest last_use (paper_2403_08837_b200.resnet.gather_zero_params). */
int cdp_resnet_zero_state(cdp_resnet *tr, int which, float *theta, uint32_t *last_use);
/* ZeRO-CDP frames: the end-of-run drain plan of this rank, n_rows x (stage, previous-occupant stage,
 * its last use kind, step offset, successor step offset) from zero.py frame_drain_plan; a drained run
 * cannot take further steps. */
int cdp_resnet_zero_drain_plan(cdp_resnet *tr, const int32_t *rows, int n_rows);
/* Theta delivery along the readers (before connect; CDP ring runs): [n_stages = world][2] = (rank this
 * rank pulls each new version of the stage from, -1 = the updater; rank that pulls it from this one, -1 =
 * none) in the rule's reader order (resnet.pull_chain).  Without it every reader pulls from the updater. */
int cdp_resnet_pull_chain(cdp_resnet *tr, const int32_t *pred_succ, int n_stages);
/* Parameter count, tensor count and (optional) per-tensor base offsets / kinds (0 conv, 1 bn, 2 fc). */
int cdp_resnet_info(cdp_resnet *tr, int64_t *n_params, int *n_tensors, int64_t *tensor_base, int32_t *tensor_kind);
int cdp_resnet_region(cdp_resnet *tr, void **base);
int cdp_resnet_ipc_handle(cdp_resnet *tr, void *handle64);
int cdp_resnet_connect(cdp_resnet *tr, void *const *regions);
void cdp_resnet_destroy(cdp_resnet *tr);
int cdp_resnet_set_params(cdp_resnet *tr, int which, const float *theta);
int cdp_resnet_get_params(cdp_resnet *tr, int which, float *theta);
int cdp_resnet_step(cdp_resnet *tr, const int32_t *perm, float lr);
/* End-to-end step: micro_batch images x (host, fp32 NHWC) and labels copied H2D inside the step. */
int cdp_resnet_step_host_batch(cdp_resnet *tr, const float *x, const int32_t *labels, float lr);
/* Pipelined end-to-end step (needs >= 2 micro-batches of dataset rows): the pinned host batch is copied
 * H2D on a copy stream into input slot `slot` (0 / 1) while the previous step computes; the step waits for
 * its copy, reads its rows, and its loss is copied back to pinned host memory.  Asynchronous: the caller
 * must not rewrite the host batch until the step has synchronised (cdp_resnet_sync). */
int cdp_resnet_step_host_batch_async(cdp_resnet *tr, const float *x, const int32_t *labels, float lr, int slot);
/* Loss of the most recent step (synchronises). */
int cdp_resnet_last_loss(cdp_resnet *tr, double *loss);
/* One real training step launched eagerly with timing events around every kernel:
 * per launch its name (name_len bytes each), algorithmic flops / bytes and duration.
 * serial != 0: all launches on one stream (clean per-kernel durations). */
int cdp_resnet_profile_step(cdp_resnet *tr, const int32_t *perm, float lr, int serial, int max_ops, char *names,
                            int name_len, double *flops, double *bytes, float *ms, int *n_ops);
int cdp_resnet_history(cdp_resnet *tr, int max, double *losses, uint32_t *flags, int *count);
int cdp_resnet_sync(cdp_resnet *tr);
int cdp_resnet_ring_error(cdp_resnet *tr, int *err);
/* out[0..5] = activation bytes, parameter-state bytes, kernels per step, tensor-core flops per step,
 * gradient scratch bytes, ZeRO-CDP state bytes received per step. */
int cdp_resnet_stats(cdp_resnet *tr, int64_t *out, int n_out);
int cdp_resnet_mark(cdp_resnet *tr, int k);
int cdp_resnet_elapsed(cdp_resnet *tr, int a, int b, float *ms);
int cdp_resnet_flush_l2(cdp_resnet *tr);
/* Device address, size and row pitch (elements; 0 = flat) of one internal buffer, for tests and
 * diagnostics after cdp_resnet_sync.  Names: "wc_hi"/"wc_lo" (index = slot * n_tensors + tensor),
 * "act_hi"/"act_lo" (activation), "y", "dy_hi", "dy_lo", "mean", "rstd", "dgamma", "dbeta" (conv
 * index), "gbuf" (0..3), "dpooled", "z", "pooled_hi", "pooled_lo", "dz_hi", "dz_lo", "theta" (0 current, 1 previous
 * slot), "region", "pool_arg" (max-pool window
 * argmax, u8 r*3+s per output element). */
int cdp_resnet_buffer(cdp_resnet *tr, const char *name, int index, void **ptr, size_t *bytes, int *ld);
/* Trace mode (create option bit 1, value 2): the executed-version record of every parameter access,
 * 8 x uint32 per record: step t, rank, unit (1-based tensor), kind (0 forward read, 1 backward read,
 * 2 update read of theta_t, 3 update's new slot), phase (0 before / 1 after the access), theta slot,
 * version tag found in the slot, 0.  Copies up to max_records (count = all recorded since the last
 * call) and clears the log.  Version tags travel with the data: set_params, updates, pulls and
 * ZeRO-CDP state copies write them (ref engine.py:92-94 records (t, i, j, v) per read). */
int cdp_resnet_trace(cdp_resnet *tr, uint32_t *records, int max_records, int *count);

/* ---- Vision Transformers (BASELINE configs[3]: ViT-B/16, 224x224), bf16 operands ------------ */
/* One worker per process, same ring / hop / pull protocol as the ResNet trainer.  Model:
 * conv patch embedding (kernel = stride = patch), class token, position embedding, `depth`
 * pre-LN blocks (LN eps 1e-6, fused qkv attention with head dim 64, GELU MLP), final LN, head
 * on the class token.  Hop units in order: patch [[W^T]; b] ([patch*patch*3 + 1][dim]), cls [dim],
 * pos [tokens][dim], per block ln1 [g | b], qkv [[W^T]; b] ([dim+1][3 dim]), proj, ln2, fc1
 * ([dim+1][mlp]), fc2 ([mlp+1][dim]), final ln, head ([dim+1][classes]); unit_stage[i] groups them
 * into world stages.  Dataset: x fp32 NHWC [n][image][image][3], labels int32.  dtype
 * CDP_DTYPE_BF16: bf16 operands, fused attention (the bench path); CDP_DTYPE_FP32: operands as
 * tf32 hi + lo pairs (3xTF32 tcgen05 products), attention as batched GEMMs with an fp32 softmax. */
typedef struct cdp_vit cdp_vit;
int cdp_vit_create_rank(int image, int patch, int dim, int depth, int heads, int mlp, int classes, int micro_batch,
                        int world, int rank, const int32_t *unit_stage, const uint8_t *stage_fresh, float momentum,
                        float weight_decay, int n_samples, const float *x, const int32_t *labels, int dtype,
                        cdp_vit **out);
/* Single-GPU cyclic CDP (BASELINE configs[3]; ref schedule.py:236-257, all workers on gpu 0):
 * n_workers micro-batches = stages on this GPU, stepped through the reference's SINGLE_GPU_CDP
 * (or SINGLE_GPU_DP) timeline.  ops[n_ops][3] = (kind 0 F / 1 B, worker 1..n, stage 1..n) in
 * timeline order (paper_2403_08837_b200/executor.compile_segment_plan); a stage task runs its
 * segments (0 = embedding, 1..depth = blocks, depth+1 = final LN + head) forward ascending /
 * backward descending.  fresh[n_workers][n_workers] is the rule table (1 = reads theta_t,
 * ref rules.py:45-51; all ones for DP).  rec_slot[n_workers][depth + 2] = activation-record slot of
 * (worker, segment) in its pool; pools[3] = embed / block / final slots (the plan's interval
 * colouring: the peak-activation claim of ref costs.py:111-115 is the pool sizes).  Gradient chain
 * S = g_1 + ... + g_n in worker order; worker n fuses the update.  probe != 0 adds a device
 * counter of live record bytes (stats out[4] = its high-water mark).  Dataset as create_rank;
 * step perms hold n_workers * micro_batch indices, worker-major. */
int cdp_vit_create_cyclic(int image, int patch, int dim, int depth, int heads, int mlp, int classes, int micro_batch,
                          int n_workers, const int32_t *unit_stage, const uint8_t *fresh, int n_ops,
                          const int32_t *ops, const int32_t *rec_slot, const int32_t *pools, float momentum,
                          float weight_decay, int probe, int n_samples, const float *x, const int32_t *labels,
                          int dtype, cdp_vit **out);
int cdp_vit_info(cdp_vit *tr, int64_t *n_params, int *n_units);
/* Trace mode (set before cdp_vit_connect): records as cdp_resnet_trace, unit = 1-based hop unit. */
int cdp_vit_set_trace(cdp_vit *tr, int on);
int cdp_vit_trace(cdp_vit *tr, uint32_t *records, int max_records, int *count);
int cdp_vit_region(cdp_vit *tr, void **base);
int cdp_vit_ipc_handle(cdp_vit *tr, void *handle64);
int cdp_vit_connect(cdp_vit *tr, void *const *regions);
void cdp_vit_destroy(cdp_vit *tr);
int cdp_vit_set_params(cdp_vit *tr, int which, const float *theta);
int cdp_vit_get_params(cdp_vit *tr, int which, float *theta);
int cdp_vit_step(cdp_vit *tr, const int32_t *perm, float lr);
int cdp_vit_step_host_batch(cdp_vit *tr, const float *x, const int32_t *labels, float lr);
int cdp_vit_profile_step(cdp_vit *tr, const int32_t *perm, float lr, int serial, int max_ops, char *names,
                         int name_len, double *flops, double *bytes, float *ms, int *n_ops);
int cdp_vit_history(cdp_vit *tr, int max, double *losses, uint32_t *flags, int *count);
int cdp_vit_sync(cdp_vit *tr);
int cdp_vit_ring_error(cdp_vit *tr, int *err);
/* out[0] activation-record bytes allocated (pool slots x record bytes), [1] parameter-state bytes,
 * [2] kernels per step, [3] tensor flops per step, [4] executed high-water mark of live record bytes
 * (probe), [5..7] bytes of one embed / block / final record, [8..10] slots per pool. */
int cdp_vit_stats(cdp_vit *tr, int64_t *out, int n_out);
int cdp_vit_mark(cdp_vit *tr, int k);
int cdp_vit_elapsed(cdp_vit *tr, int a, int b, float *ms);
int cdp_vit_flush_l2(cdp_vit *tr);
/* Theta delivery along the readers, as cdp_resnet_pull_chain (before connect). */
int cdp_vit_pull_chain(cdp_vit *tr, const int32_t *pred_succ, int n_stages);
/* Fused multi-head attention (csrc/attn_kernels.cuh) on caller-owned device buffers: bf16 token-major
 * qkv [B*T][qkv_ld] (Q | K | V blocks of H*64 columns, head h at +h*64), O [B*T][o_ld], lse fp32
 * [B*H*T]; backward != 0 also writes dQ | dK | dV into dqkv from dO.  T <= 256, head dim 64, scale 1/8.
 * No reference counterpart (the reference trains no attention model): the ViT trainer's layer compute
 * (north_star (4)), exported for its parity tests. */
int cdp_attention(const void *qkv, int64_t qkv_ld, const void *dout, int64_t dout_ld, int T, int H, int B, void *o,
                  int64_t o_ld, float *lse, void *dqkv, int64_t dqkv_ld, int backward);


/* ---- tensor-core GEMM self-test (parity tests of the tcgen05 kernel) --- */
/* D[m][n] = sum_s A_s . B_s.  kind 0 = bf16, 1 = fp32/tf32.  A K-major:
 * A[m*lda+k], MN-major: A[k*lda+m]; B K-major: B[n*ldb+k], MN-major:
 * B[k*ldb+n].  Device pointers; stream may be NULL. */
int cdp_test_gemm(int kind, int a_mn, int b_mn, int bn, int M, int N, int K, int n_seg, const void *const *a_ptrs,
                  int lda, const void *const *b_ptrs, int ldb, float *d, int ldd, int splits, float *ws,
                  int *counters, void *stream);

#ifdef __cplusplus
}
#endif
#endif /* CDP_B200_H */
