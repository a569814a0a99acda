#!/usr/bin/env python
"""CDP training-step benchmark on B200 (contract: DESIGN.md §8 Measurement).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
                    [--model resnet18|resnet50|mlp] [--dtype bf16|fp32] [--rule cdp-v2|cdp-v1|dp]
    torchrun --nproc-per-node N bench.py --gpus N ...

Headline workload (default, --model resnet50) = BASELINE configs[2], the north-star target:
ResNet-50 (torchvision v1.5 layout) on ImageNet-shaped synthetic data (224x224x3, 1000 classes),
CDP-v2, ONE micro-batch of B = 128 per GPU, N = micro-batches = stages = GPUs (FLOP-balanced
contiguous tensor groups), SGD lr 0.05 momentum 0.9, bf16 operands / fp32 master state.  One step =
the whole job's training step: every rank's forward + backward, the per-tensor gradient hops
rank -> rank+1 over peer memory fused into the weight-gradient GEMM epilogues, the fused update on
the last rank, the parameter pulls; one CUDA graph per rank, no collective.  Per-GPU work is fixed
as N grows (weak scaling).

`value` = samples/s of the device-timed step (CUDA events on each rank's launch stream around each
graph launch, inputs resident in HBM, L2 flushed by a 256 MiB memset before every timed step, max
over ranks); `e2e` = the same through the public API with the step's images / labels copied H2D
from pinned host memory inside every step and the loss read back every step.  `roofline` = the
dominant tensor-core kernel class of a serialised instrumented step (algorithmic conv flops /
event-timed duration) against MEASURED_PEAKS.json.  N > 1 adds `exposed_comm` (ring step minus the
compute-only step of the same per-rank work) and `p2p` (hop / pull bytes per rank, GB/s in the
kernels that move them).  At N = 1 the line also carries `resnet18` (configs[1] shape),
`vit_b16_single_gpu_cdp` (configs[3]: ViT-B/16, 4 and 12 sequential micro-batches on one GPU,
CDP-v2 vs DP with the device-measured activation high-water marks) and `single_gpu_cdp` (configs[0]:
the reference's own CPU-runnable MLP case with its CPU time).  `cpu_baseline` / `--impl reference`:
the reference has no ResNet, so the CPU arm is the oracle port (oracle/resnet_torch.py:
the reference's `_advance` semantics over torch-CPU float64 autograd) on all host cores, on a
bounded sample of the same workload.
"""

from __future__ import annotations

import argparse
import json
import os
import statistics
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

with open(os.path.join(ROOT, "BASELINE.json")) as _fh:
    METRIC = json.load(_fh)["metric"]
UNIT = "samples/s"
RN_MB = 128
RN_LR, RN_MOMENTUM = 0.05, 0.9
DEEP_DIMS = (3072,) + (256,) * 7 + (10,)
MB = 128
CONFIG1 = dict(n=4, micro_batch_size=32, seed=0, width=256, in_dim=3072, out_dim=10, loss_kind="xent")
LR, MOMENTUM = 0.05, 0.9


def dist_env():
    return int(os.environ.get("WORLD_SIZE", "1")), int(os.environ.get("RANK", "0")), int(os.environ.get("LOCAL_RANK", "0"))


def make_deep_task(n: int, seed: int = 0):
    """Synthetic CIFAR-shaped data for the deep MLP, generated like the reference's make_mlp_task
    (x ~ N(0,1) from default_rng([seed, 0xB0]); labels = argmax of a teacher from [seed, 0xB1])."""
    from paper_2403_08837_b200.training.models import StageMlp, ToyTask

    model = StageMlp(dims=DEEP_DIMS, loss_kind="xent")
    rng = np.random.default_rng([seed, 0xB0])
    x = rng.normal(0.0, 1.0, size=(n * MB, DEEP_DIMS[0]))
    y = np.argmax(model.forward(model.init_params(np.random.default_rng([seed, 0xB1])), x), axis=1).astype(np.int64)
    return ToyTask(model, x, y, n, MB, seed)


def workload_name(n, rule, dtype):
    return (f"CDP one micro-batch per GPU: 8-layer MLP 3072-256x7-10 in {n} stage(s), B={MB}/GPU, xent, "
            f"{rule}, {dtype}, SGD lr {LR} momentum {MOMENTUM} (stage-MLP stand-in for configs[1])")


def peak_hbm():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    try:
        with open(p) as fh:
            return float(json.load(fh)["hbm_gbs"]), "measured"
    except Exception:
        return 6650.0, "fallback"


# ----------------------------------------------------------------------------- clocks
class ClockSampler:
    """nvml samples of SM clock and throttle reasons, ~1 kHz, during the timed region."""

    REASONS = {0x4: "sw_power_cap", 0x8: "hw_slowdown", 0x20: "sw_thermal_slowdown", 0x40: "hw_thermal_slowdown",
               0x80: "hw_power_brake_slowdown", 0x2: "applications_clocks_setting", 0x10: "sync_boost"}

    def __init__(self, index=0):
        self.samples, self.reasons, self.ok, self.max_mhz = [], set(), False, None
        try:
            import pynvml

            pynvml.nvmlInit()
            self.nv = pynvml
            self.h = pynvml.nvmlDeviceGetHandleByIndex(index)
            self.max_mhz = pynvml.nvmlDeviceGetMaxClockInfo(self.h, pynvml.NVML_CLOCK_SM)
            self.ok = True
        except Exception:
            pass
        self._stop = threading.Event()

    def _run(self):
        while not self._stop.is_set():
            try:
                self.samples.append(self.nv.nvmlDeviceGetClockInfo(self.h, self.nv.NVML_CLOCK_SM))
                r = self.nv.nvmlDeviceGetCurrentClocksEventReasons(self.h)
                self.reasons.update(name for bit, name in self.REASONS.items() if r & bit)
            except Exception:
                pass
            time.sleep(0.001)

    def __enter__(self):
        if self.ok:
            self._t = threading.Thread(target=self._run, daemon=True)
            self._t.start()
        return self

    def __exit__(self, *a):
        self._stop.set()
        if self.ok:
            self._t.join()

    def summary(self):
        return {"sm_mhz": statistics.median(self.samples) if self.samples else None, "sm_max_mhz": self.max_mhz,
                "reasons": sorted(self.reasons), "samples": len(self.samples)}


# ----------------------------------------------------------------------------- CPU reference
def _ref_job(args):
    dims, theta, x, labels = args
    from oracle import kernels as OK

    mod = OK.load_reference_kernels()
    if mod is None:
        return OK.mlp_value_grad(dims, theta, x, None, labels, 1)
    return mod.mlp_value_grad(dims, theta, x, None, labels, 1)


def cpu_reference(task, fresh, steps, warmup, procs):
    """The reference's CPU step (ref engine.py:66-116 restated in oracle/engine.py) with its compiled
    kernel (oracle/_ref) per micro-batch; `procs` > 1 evaluates the micro-batches in parallel processes."""
    from oracle import engine as OE
    from oracle import kernels as OK

    kind = "reference" if OK.load_reference_kernels() is not None else "port"
    sizes = task.model.stage_sizes
    dims = task.model.dims
    cur = [p.copy() for p in task.init_params()]
    prev = [p.copy() for p in cur]
    vel = [np.zeros_like(p) for p in cur]
    pool = None
    if procs > 1:
        import multiprocessing as mp

        pool = mp.get_context("fork").Pool(procs)

    def one(t):
        nonlocal cur, prev
        batches = task.micro_batches(t)
        params = [[cur[j] if (fresh is None or fresh[i][j]) else prev[j] for j in range(len(cur))]
                  for i in range(task.n)]
        jobs = [(dims, np.concatenate(params[i]), batches[i][0], batches[i][1].astype(np.int64)) for i in range(task.n)]
        res = pool.map(_ref_job, jobs) if pool else [_ref_job(j) for j in jobs]
        it = iter(res)

        def gfn(_p, _x, _y):
            loss, g = next(it)
            return loss, OE.split(g, sizes)

        new, _ = OE.advance(task, cur, prev, t, batches, LR, fresh, MOMENTUM, vel, grads_fn=gfn)
        prev, cur = cur, new

    for t in range(1, warmup + 1):
        one(t)
    t0 = time.perf_counter()
    for t in range(warmup + 1, warmup + steps + 1):
        one(t)
    dt = (time.perf_counter() - t0) / steps
    if pool:
        pool.close()
    return task.n * task.micro_batch_size / dt, dt * 1e3, kind


def expanded_fresh(rule, n, layer_stage):
    if rule is None:
        return None
    return [[rule.reads_fresh(i, layer_stage[l]) for l in range(len(layer_stage))] for i in range(1, n + 1)]


# ----------------------------------------------------------------------------- our arm
def run_ours(args, ws, rank, local):
    import torch

    torch.cuda.set_device(local)
    from paper_2403_08837_b200.device import DeviceMlpTrainer
    from paper_2403_08837_b200.dist import exchange_handles, resolve
    from paper_2403_08837_b200.executor import layer_stages

    task = make_deep_task(ws)
    allreduce = args.rule == "dp-allreduce"
    rule = None if allreduce else resolve(args.rule, ws)
    ls = layer_stages(len(DEEP_DIMS) - 1, ws)
    tr = DeviceMlpTrainer.for_rank(DEEP_DIMS, MB, ws, rank, 1, rule, dtype=args.dtype, momentum=MOMENTUM,
                                   inputs=task.inputs, targets=task.targets, layer_stage=ls, allreduce=allreduce)
    tr.set_params(np.concatenate(task.init_params()), which=-1)
    if ws > 1:
        tr.connect_ipc(exchange_handles(tr.ipc_handle()))
        torch.distributed.barrier()  # every rank captured its graphs before any step spins on a peer
    else:
        tr.connect([tr.region()])
    perms = [task.permutation(t)[rank * MB:(rank + 1) * MB] for t in range(1, args.warmup + args.steps + 2)]
    if allreduce:  # DP baseline: NCCL all-reduce of the gradient on the trainer stream, then the update
        ext = torch.cuda.ExternalStream(tr.stream_handle())
        grad = tr.partial_tensor()
        plain_step = tr.step

        def dp_reduce_update():
            if ws > 1:
                with torch.cuda.stream(ext):
                    torch.distributed.all_reduce(grad)
            tr.apply_update()

        def dp_step(perm, lr):
            plain_step(perm, lr)
            dp_reduce_update()

        tr.step = dp_step
    for t in range(args.warmup):
        tr.step(perms[t], LR)
    tr.sync()
    if ws > 1:
        torch.distributed.barrier()
    K = args.steps
    with ClockSampler(local) as clk:
        for k in range(K):
            tr.flush_l2()
            tr.mark(2 * k)
            tr.step(perms[args.warmup + k], LR)
            tr.mark(2 * k + 1)
        tr.sync()
    if tr.ring_error():
        raise RuntimeError(f"rank {rank}: ring protocol timed out")
    ms = float(np.mean([tr.elapsed(2 * k, 2 * k + 1) for k in range(K)]))
    if ws > 1:
        t = torch.tensor([ms], device="cuda")
        torch.distributed.all_reduce(t, op=torch.distributed.ReduceOp.MAX)
        ms = float(t.item())
    losses, flags = tr.history(K + args.warmup)
    assert np.all(np.isfinite(losses)) and not flags.any(), "non-finite step in the timed region"
    value = ws * MB / (ms / 1e3)
    stats = tr.stats()

    # ---- e2e: public API, pinned host micro-batch copied H2D every step, loss read back every step
    x_pin = torch.empty((MB, DEEP_DIMS[0]), dtype=torch.float32, pin_memory=True)
    y_pin = torch.empty((MB,), dtype=torch.int32, pin_memory=True)
    host = [(task.inputs[p].astype(np.float32), task.targets[p].astype(np.int32)) for p in perms[:K + 2]]
    e2e_ms = []
    if ws > 1:
        torch.distributed.barrier()
    for k in range(K + 2):
        x_pin.numpy()[:] = host[k][0]
        y_pin.numpy()[:] = host[k][1]
        tr.flush_l2()
        tr.mark(0)
        tr.step_host_batch_ptr(x_pin.data_ptr(), y_pin.data_ptr(), LR)
        if allreduce:
            dp_reduce_update()
        tr.last()
        tr.mark(1)
        if k >= 2:
            e2e_ms.append(tr.elapsed(0, 1))
    e2e = float(np.mean(e2e_ms))
    if ws > 1:
        t = torch.tensor([e2e], device="cuda")
        torch.distributed.all_reduce(t, op=torch.distributed.ReduceOp.MAX)
        e2e = float(t.item())
    h2d = MB * DEEP_DIMS[0] * 4 + MB * 4 + 16 + MB * 4
    d2h = 8 + 16

    # ---- roofline: layer-1 weight-grad GEMM with the fused hop (update when N = 1)
    op = tr.op_index(1, rank + 1, 1)
    if allreduce:
        mode = "grad"
    kms = []
    for _ in range(20):
        tr.flush_l2()
        kms.append(tr.time_op(op, 4, -1))
    k_ms = float(np.median(kms))
    p1 = DEEP_DIMS[0] * DEEP_DIMS[1] + DEEP_DIMS[1]
    esz = 2 if args.dtype == "bf16" else 8
    if not allreduce:
        mode = "only" if ws == 1 else ("first" if rank == 0 else "last" if rank == ws - 1 else "mid")
    per_param = {"first": 4, "mid": 8, "last": 20 + esz, "only": 16 + esz, "grad": 4}[mode]
    alg = p1 * per_param + MB * (DEEP_DIMS[0] + DEEP_DIMS[1]) * (2 if args.dtype == "bf16" else 8)
    peak, src = peak_hbm()
    achieved = alg / (k_ms / 1e3) / 1e9
    traffic = None
    tp = os.path.join(ROOT, "profiles", "round1_wgrad_hop_traffic.json")
    if os.path.exists(tp):
        with open(tp) as fh:
            traffic = (json.load(fh).get(f"{args.dtype}-{mode}") or {}).get("dram_bytes_per_launch")

    out = {
        "metric": METRIC, "value": round(value, 1), "unit": UNIT, "n_gpus": ws, "steps": K, "warmup": args.warmup,
        "ms_per_step": round(ms, 5), "higher_is_better": True, "scaling": "weak", "vs_baseline": None,
        "dtype": args.dtype, "data": "synthetic (numpy PCG64, teacher-labelled, reference make_mlp_task recipe)",
        "config": {"workload": workload_name(ws, args.rule, args.dtype), "global_batch": ws * MB, "micro_batch": MB,
                   "stages": ws, "layers": len(DEEP_DIMS) - 1, "rule": args.rule,
                   "parallelism": f"cdp{ws} (one process per GPU, P2P hop ring, fused update on rank {ws - 1})",
                   "l2": "flushed (256 MiB memset) before every timed step"},
        "e2e": {"value": round(ws * MB / (e2e / 1e3), 1), "unit": UNIT, "h2d_bytes_per_step": h2d,
                "d2h_bytes_per_step": d2h, "ms_per_step": round(e2e, 5)},
        "gpu_launches": (stats["kernels_per_step"] + (len(DEEP_DIMS) - 1 if allreduce else 0)) * K,
        "roofline": {"bound": "hbm", "kernel": f"layer-1 wgrad GEMM + fused {mode} hop (gemm_tc_kernel<EpiWgrad>)",
                     "achieved": round(achieved, 1), "peak": peak, "peak_source": src, "unit": "GB/s",
                     "frac": round(achieved / peak, 4), "traffic": traffic, "algorithmic_bytes_per_launch": alg,
                     "launch_us": round(k_ms * 1e3, 2)},
        "activation_bytes": {"per_gpu": stats["activation_bytes"], "sum_over_gpus": stats["activation_bytes"] * ws},
        "clocks": clk.summary(),
    }
    tr.close()
    return out, task, rule, ls


# ----------------------------------------------------------------------------- ResNet arm
def resnet_cfg(model):
    from paper_2403_08837_b200.resnet import RESNET18, RESNET50

    if model == "resnet18":
        return dict(RESNET18), 32, 10
    return dict(RESNET50), 224, 1000


VIT_MB = 32  # BASELINE configs[3] / SURVEY §8d: ViT-B/16, B = 32


def make_trainer(args, model, ws, rank, rule, allreduce, zero):
    """(trainer, micro-batch, image side, classes, dataset x, labels) for a bench model.  With ws = 1 and
    rule = None the trainer is the compute-only twin of a ring rank (same per-GPU work, fused update,
    no peer reads / waits / pulls): the baseline of `exposed_comm_ms`."""
    from paper_2403_08837_b200.resnet import DeviceResNet, init_params, layer_specs, synthetic_images

    if model == "vit_b16":
        from paper_2403_08837_b200.vit import VIT_B16, DeviceVit, vit_init

        if allreduce or zero:
            raise SystemExit("vit_b16: --rule dp-allreduce / --zero are built for the ResNets")
        B = VIT_MB
        x, y = synthetic_images(2 * B * ws, seed=0, hw=224, classes=1000)
        tr = DeviceVit(VIT_B16, B, ws, rank, rule, RN_MOMENTUM, inputs=x, labels=y, dtype=args.dtype)
        tr.set_params(vit_init(VIT_B16, seed=0), -1)
        return tr, B, 224, 1000, x, y
    cfg, hw, classes = resnet_cfg(model)
    B = RN_MB
    x, y = synthetic_images(2 * B * ws, seed=0, hw=hw, classes=classes)
    specs = layer_specs(cfg["widths"], cfg["depths"], 3, hw, cfg["block"], cfg["stem"], classes)
    tr = DeviceResNet(cfg["widths"], cfg["depths"], B, ws, rank, rule, args.dtype, RN_MOMENTUM, inputs=x, labels=y,
                      classes=classes, image_hw=hw, block=cfg["block"], stem=cfg["stem"], zero=zero,
                      dp_allreduce=allreduce)
    tr.set_params(init_params(specs, seed=0), -1)
    return tr, B, hw, classes, x, y


def peak_tensor():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    try:
        with open(p) as fh:
            return float(json.load(fh)["bf16_tflops"]), "measured (burst)"
    except Exception:
        return 2250.0, "fallback (spec dense bf16)"


def kernel_table(ops):
    """Group an instrumented step's launches by kernel class: {name: [launches, ms, flops, bytes]}."""
    agg = {}
    for name, fl, by, ms in ops:
        a = agg.setdefault(name, [0, 0.0, 0.0, 0.0])
        a[0] += 1
        a[1] += ms
        a[2] += fl
        a[3] += by
    return agg


def run_resnet(args, ws, rank, local, model, steps, warmup, e2e=True):
    import torch

    from paper_2403_08837_b200.dist import exchange_handles, resolve
    from paper_2403_08837_b200.resnet import DeviceResNet, init_params, layer_specs, synthetic_images

    torch.cuda.set_device(local % torch.cuda.device_count())  # (ranks may share a GPU in tests)
    allreduce = args.rule == "dp-allreduce"
    rule = None if allreduce else resolve(args.rule, ws)
    zero = bool(getattr(args, "zero", False)) and ws > 1
    tr, B, hw, classes, x, y = make_trainer(args, model, ws, rank, rule, allreduce, zero)
    n_data = x.shape[0]
    if ws > 1:
        tr.connect_ipc(exchange_handles(tr.ipc_handle()))
        torch.distributed.barrier()  # every rank captured its graphs before any step spins on a peer
    else:
        tr.connect([tr.region()])
    perms = [np.random.default_rng([0, t]).permutation(n_data)[rank * B:(rank + 1) * B]
             for t in range(1, warmup + steps + 8)]
    if allreduce:  # DP baseline: NCCL all-reduce of the flat gradient on the trainer stream, then the update
        ext = torch.cuda.ExternalStream(tr.stream_handle())
        grad = tr.partial_tensor()

        def reduce_update():
            if ws > 1:
                with torch.cuda.stream(ext):
                    torch.distributed.all_reduce(grad)
            tr.apply_update()
    else:
        def reduce_update():
            pass

    def do_step(perm):
        tr.step(perm, RN_LR)
        reduce_update()

    def settle():  # ZeRO-CDP: publish the next step's forwards other ranks' last step waits for
        tr.zero_drain()
        tr.sync()

    frames = bool(getattr(tr, "zero_frames", False))
    for t in range(warmup):
        do_step(perms[t])
    # ZeRO-CDP state frames: a drain ends the run (the last states move into next-step forward frames) and a
    # rank cannot synchronise mid-run, so warm-up and timed steps run back to back (the per-step device
    # events time each step) and the e2e loop / instrumented step (both synchronise per step) are skipped
    if not frames:
        settle()
    if ws > 1:
        torch.distributed.barrier()
    with ClockSampler(local) as clk:
        for k in range(steps):
            tr.flush_l2()
            tr.mark(2 * k)
            do_step(perms[warmup + k])
            tr.mark(2 * k + 1)
        settle()
    if tr.ring_error():
        raise RuntimeError(f"rank {rank}: ring protocol timed out")
    ms = float(np.mean([tr.elapsed(2 * k, 2 * k + 1) for k in range(steps)]))
    if ws > 1:
        t = torch.tensor([ms], device="cuda")
        torch.distributed.all_reduce(t, op=torch.distributed.ReduceOp.MAX)
        ms = float(t.item())
    losses, flags = tr.history(steps + warmup)
    assert np.all(np.isfinite(losses)) and not flags.any(), "non-finite step in the timed region"
    st = tr.stats()
    P = tr.P
    out = {"value": round(ws * B / (ms / 1e3), 1), "ms_per_step": round(ms, 4), "clocks": clk.summary(),
           "losses_first_last": [round(float(losses[0]), 5), round(float(losses[-1]), 5)],
           "activation_bytes": {"per_gpu": st["activation_bytes"], "sum_over_gpus": st["activation_bytes"] * ws},
           "param_state_bytes": st["param_state_bytes"], "gpu_launches": st["kernels_per_step"] * steps,
           "tensor_flops_per_step": st["tensor_flops_per_step"],
           "zero_state_bytes_per_step": st.get("zero_state_bytes_per_step", 0),
           "tensor_tflops_per_s": round(st["tensor_flops_per_step"] / (ms / 1e3) / 1e12, 1)}
    # ---- e2e: public API, pinned host images copied H2D every step, loss read back every step
    if e2e and frames:
        out["e2e"] = {"value": None, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0,
                      "note": "ZeRO-CDP state frames: a run cannot be synchronised mid-way (see run_resnet)"}
    elif e2e:
        # pinned host batches (a ring of 4 distinct batches, filled before the timed region); every step
        # copies its batch H2D on the copy stream while the previous step computes (two input slots) and
        # copies its loss back D2H; device time from the first copy to the last loss / steps
        ring = 4
        x_pins = [torch.empty((B, hw, hw, 3), dtype=torch.float32, pin_memory=True) for _ in range(ring)]
        y_pins = [torch.empty((B,), dtype=torch.int32, pin_memory=True) for _ in range(ring)]
        for k in range(ring):
            x_pins[k].numpy()[:] = x[perms[k]]
            y_pins[k].numpy()[:] = y[perms[k]]
        ke = min(steps, 20) + 2
        pipelined = hasattr(tr, "step_host_batch_async")  # ResNets; the ViT copies on its step stream

        def host_step(k):
            if pipelined:
                tr.step_host_batch_async(x_pins[k % ring].data_ptr(), y_pins[k % ring].data_ptr(), RN_LR, k % 2)
            else:
                tr.step_host_batch_ptr(x_pins[k % ring].data_ptr(), y_pins[k % ring].data_ptr(), RN_LR)

        host_step(0)  # warm the copy path
        tr.sync()
        if ws > 1:
            torch.distributed.barrier()
        tr.mark(0)
        for k in range(ke):
            tr.flush_l2()
            host_step(k)
            reduce_update()
        tr.mark(1)
        tr.sync()
        losses_e, flags_e = tr.history(ke)
        assert np.all(np.isfinite(losses_e)) and not flags_e.any()
        e = tr.elapsed(0, 1) / ke
        if ws > 1:
            t = torch.tensor([e], device="cuda")
            torch.distributed.all_reduce(t, op=torch.distributed.ReduceOp.MAX)
            e = float(t.item())
        out["e2e"] = {"value": round(ws * B / (e / 1e3), 1), "unit": UNIT,
                      "h2d_bytes_per_step": B * hw * hw * 3 * 4 + B * 4 + 16 + B * 4,
                      "d2h_bytes_per_step": 8 if pipelined else 0,
                      "ms_per_step": round(e, 4),
                      "how": ("public API step_host_batch_async: every step copies its pinned host batch H2D (copy "
                              "stream, two input slots: overlaps the previous step) and its loss D2H; device time "
                              "from before the first copy to after the last step / steps, L2 flushed every step"
                              if pipelined else
                              "public API step_host_batch: every step copies its pinned host batch H2D on the step "
                              "stream before the step (no overlap; losses stay in the device history); device time "
                              "from before the first copy to after the last step / steps, L2 flushed every step")}
    # ---- per-kernel breakdown: one serialised instrumented (real) step
    if frames:
        out["kernel_breakdown"] = None
        out["roofline"] = None
        out["serial_step_ms"] = None
        out["p2p"] = {"zero_state_bytes_per_rank0": int(st.get("zero_state_bytes_per_step", 0)),
                      "note": "ZeRO-CDP state frames: no instrumented step (see above)"}
    else:
        if ws > 1:
            torch.distributed.barrier()
        ops = tr.profile_step(perms[warmup + steps], RN_LR, serial=ws == 1)
        reduce_update()
        settle()
        agg = kernel_table(ops)
        tot = sum(a[1] for a in agg.values())
        gemm = {k: a for k, a in agg.items() if a[2] > 0}
        dom = max(gemm, key=lambda k: gemm[k][1])
        d = gemm[dom]
        peak, src = peak_tensor()
        achieved = d[2] / (d[1] / 1e3) / 1e12
        # the class's bound from its arithmetic intensity (algorithmic flops / algorithmic HBM bytes, both
        # recorded per launch by the trainer) against the ridge point of the measured peaks: the 1x1 convs
        # of ResNet-50 (K = 64..512) sit far below it and are judged against HBM bandwidth
        hbm, hsrc = peak_hbm()
        ridge = peak * 1e12 / (hbm * 1e9)
        ai = d[2] / d[3] if d[3] > 0 else float("inf")
        # DRAM bytes per launch of the same class from an ncu capture of one serialised step
        # (tools/step_traffic.py; bf16 only)
        traffic = None
        tp = os.path.join(ROOT, "profiles", "r2_step_traffic.json")
        if not os.path.exists(tp):
            tp = os.path.join(ROOT, "profiles", "r1_step_traffic.json")
        if os.path.exists(tp) and args.dtype == "bf16":
            with open(tp) as fh:
                traffic = ((json.load(fh).get(model) or {}).get(dom) or {}).get("dram_bytes_per_launch")
        out["roofline"] = {"bound": "tensor", "kernel": f"{dom} (gemm_pk_kernel, tcgen05 + TMA; {d[0]} launches)",
                           "achieved": round(achieved, 1), "peak": peak, "peak_source": src, "unit": "TFLOP/s",
                           "frac": round(achieved / peak, 4), "traffic": traffic,
                           "algorithmic_flops_per_launch": round(d[2] / d[0]),
                           "algorithmic_bytes_per_launch": round(d[3] / d[0]),
                           "arithmetic_intensity_flop_per_byte": round(ai, 1), "ridge_flop_per_byte": round(ridge, 1),
                           "launch_us": round(d[1] / d[0] * 1e3, 2), "share_of_serial_step": round(d[1] / tot, 3)}
        if ai < ridge:
            gbs = d[3] / (d[1] / 1e3) / 1e9
            out["roofline"].update({"bound": "hbm", "achieved": round(gbs, 1), "peak": hbm, "peak_source": hsrc,
                                    "unit": "GB/s", "frac": round(gbs / hbm, 4),
                                    "tensor_tflops": round(achieved, 1), "tensor_frac": round(achieved / peak, 4)})
        # ---- P2P traffic of this step (bytes per rank, one micro-batch per GPU): the gradient hop reads the
        # previous rank's partial sum S (4 B / param, ranks 2..N, fused into the weight-gradient epilogues);
        # every reader pulls the versions it reads from the updater (4 B / param, ranks 1..N-1); ZeRO-CDP
        # copies states instead of pulling.  GB/s = those bytes / the event-timed durations of the kernels
        # that move them on this rank (the hop-fused GEMMs also compute, so theirs is a lower bound).
        if ws > 1:
            hop_b = 4 * P if rank > 0 else 0
            pull_b = 0 if (rank == ws - 1 or zero or allreduce) else 4 * P
            zero_b = int(st.get("zero_state_bytes_per_step", 0))
            hop_ms = sum(a[1] for k, a in agg.items() if "hop" in k and "wait" not in k)
            pull_ms = sum(a[1] for k, a in agg.items() if k in ("pull", "zero_copy"))
            vals = torch.tensor([hop_b, pull_b, zero_b, hop_ms, pull_ms], dtype=torch.float64, device="cuda")
            allv = [torch.zeros_like(vals) for _ in range(ws)]
            torch.distributed.all_gather(allv, vals)
            allv = [v.cpu().numpy() for v in allv]
            out["p2p"] = {
                "grad_hop_read_bytes_per_rank": [int(v[0]) for v in allv],
                "param_pull_read_bytes_per_rank": [int(v[1]) for v in allv],
                "zero_state_bytes_per_rank": [int(v[2]) for v in allv],
                "bytes_per_step_all_ranks": int(sum(v[0] + v[1] + v[2] for v in allv)),
            "pull_sources": ("reader chain (csrc/rank_common.cuh): the updater and every reader serve at most one "
                             "copy of each version, 4 B / param per step"
                             if getattr(tr, "pull_chain", None) is not None else
                             "every reader pulls from the updater: (N-1) x 4 B / param of updater egress"),
                "grad_gbs_in_hop_kernels_rank1": round(allv[1][0] / (allv[1][3] / 1e3) / 1e9, 1) if allv[1][3] else None,
                "pull_gbs_rank0": round((allv[0][1] + allv[0][2]) / (allv[0][4] / 1e3) / 1e9, 1) if allv[0][4] else None,
                "note": "peer HBM over NVLink when ranks sit on different GPUs; same-GPU ranks (tests) read local HBM"}
        else:
            out["p2p"] = {"bytes_per_step_all_ranks": 0, "note": "one GPU: no peer traffic (the hop is local)"}
        out["kernel_breakdown"] = {
            k: {"launches": a[0], "ms": round(a[1], 4), "share": round(a[1] / tot, 3),
                **({"tflops": round(a[2] / (a[1] / 1e3) / 1e12, 1)} if a[2] else {}),
                **({"gbs": round(a[3] / (a[1] / 1e3) / 1e9, 1)} if a[3] or not a[2] else {})}
            for k, a in sorted(agg.items(), key=lambda kv: -kv[1][1])}
        out["serial_step_ms"] = round(tot, 4)
    tr.close()
    # ---- exposed gradient communication (N > 1): full ring step - compute-only step of the same rank work
    if ws > 1 and not allreduce:
        from paper_2403_08837_b200.dist import resolve as _resolve

        co, *_ = make_trainer(args, model, 1, 0, _resolve(args.rule, 1), False, False)
        co.connect([co.region()])
        cperms = [np.random.default_rng([0, t]).permutation(2 * B)[:B] for t in range(warmup + steps)]
        for t in range(warmup):
            co.step(cperms[t], RN_LR)
        co.sync()
        torch.distributed.barrier()
        for k in range(steps):
            co.flush_l2()
            co.mark(2 * k)
            co.step(cperms[warmup + k], RN_LR)
            co.mark(2 * k + 1)
        co.sync()
        cms = float(np.mean([co.elapsed(2 * k, 2 * k + 1) for k in range(steps)]))
        co.close()
        t = torch.tensor([cms], device="cuda")
        torch.distributed.all_reduce(t, op=torch.distributed.ReduceOp.MAX)
        cms = float(t.item())
        out["exposed_comm"] = {"compute_only_ms_per_step": round(cms, 4),
                               "exposed_comm_ms": round(ms - cms, 4), "exposed_frac": round((ms - cms) / ms, 4),
                               "how": "max-over-ranks step of the ring minus max-over-ranks step of the same "
                                      "per-rank work as a one-GPU trainer (fused update, no peer reads / waits / "
                                      "pulls), both device-timed with L2 flushed"}
    elif ws == 1:
        out["exposed_comm"] = {"exposed_comm_ms": 0.0, "note": "one GPU: no gradient communication"}
    return out


def run_resnet_variant(args, ws, rank, local, model, steps, warmup, mode):
    """Timed steps of one comparison variant at the same N, shape and per-GPU micro-batch (all ranks):
    "dp-allreduce" (DP: NCCL all-reduce of the flat gradient + update), "zero-cdp" (ZeRO-CDP: P2P state
    passing along the reference holder chain) or "zero-dp" (ZeRO-DP: per-stage owner broadcast +
    gradient reduce to the owner, resnet.ZeroDpRank).  Device-timed (trainer stream events), L2 flushed,
    max over ranks."""
    import argparse as _ap

    import torch

    from paper_2403_08837_b200.dist import exchange_handles, resolve

    allreduce = mode in ("dp-allreduce", "zero-dp")
    zero = mode == "zero-cdp"
    a2 = _ap.Namespace(**vars(args))
    a2.rule = "dp-allreduce" if allreduce else "cdp-v2"
    rule = None if allreduce else resolve("cdp-v2", ws)
    tr, B, hw, classes, x, y = make_trainer(a2, model, ws, rank, rule, allreduce, zero)
    if ws > 1:
        tr.connect_ipc(exchange_handles(tr.ipc_handle()))
        torch.distributed.barrier()  # every rank captured its graphs before any step spins on a peer
    else:
        tr.connect([tr.region()])
    perms = [np.random.default_rng([0, t]).permutation(x.shape[0])[rank * B:(rank + 1) * B]
             for t in range(1, warmup + steps + 2)]
    zd = None
    if mode == "zero-dp":
        from paper_2403_08837_b200.resnet import ZeroDpRank

        zd = ZeroDpRank(tr)
    elif mode == "dp-allreduce":
        ext = torch.cuda.ExternalStream(tr.stream_handle())
        grad = tr.partial_tensor()

    def do_step(perm):
        if zd is not None:
            zd.step(perm, RN_LR)
            return
        tr.step(perm, RN_LR)
        if mode == "dp-allreduce":
            if ws > 1:
                with torch.cuda.stream(ext):
                    torch.distributed.all_reduce(grad)
            tr.apply_update()

    for t in range(warmup):
        do_step(perms[t])
    if not getattr(tr, "zero_frames", False):  # (state frames: a drain ends the run, see run_resnet)
        tr.zero_drain()
        tr.sync()
    if ws > 1:
        torch.distributed.barrier()
    for k in range(steps):
        tr.flush_l2()
        tr.mark(2 * k)
        do_step(perms[warmup + k])
        tr.mark(2 * k + 1)
    tr.zero_drain()
    tr.sync()
    if tr.ring_error():
        raise RuntimeError(f"rank {rank}: ring protocol timed out ({mode})")
    ms = float(np.mean([tr.elapsed(2 * k, 2 * k + 1) for k in range(steps)]))
    st = tr.stats()
    state_b = zd.bytes_per_step if zd is not None else int(st.get("zero_state_bytes_per_step", 0))
    if ws > 1:
        t = torch.tensor([ms], device="cuda")
        torch.distributed.all_reduce(t, op=torch.distributed.ReduceOp.MAX)
        ms = float(t.item())
        v = torch.tensor([float(state_b)], device="cuda")
        allv = [torch.zeros_like(v) for _ in range(ws)]
        torch.distributed.all_gather(allv, v)
        state_b = [int(a.item()) for a in allv]
    tr.close()
    return {"value": round(ws * B / (ms / 1e3), 1), "unit": UNIT, "ms_per_step": round(ms, 4),
            "state_bytes_per_step_per_rank": state_b, "param_state_bytes_per_rank": st["param_state_bytes"]}


def vit_single_gpu(n, steps, warmup, profile=False):
    """BASELINE configs[3]: ViT-B/16 224x224, n sequential micro-batches of VIT_MB on ONE GPU, stepped
    through the reference's SINGLE_GPU_CDP (cdp-v2) and SINGLE_GPU_DP timelines by the cyclic executor
    (DeviceVit.single_gpu).  Peak activation = the device's live-record high-water mark (a counter
    updated around every record acquire / release in the captured step), cross-checked against the
    allocator (cudaMemGetInfo delta of creating the trainer) and the plan's time-resolved peak."""
    import torch

    from paper_2403_08837_b200.resnet import synthetic_images
    from paper_2403_08837_b200.rules import rule_by_name
    from paper_2403_08837_b200.vit import VIT_B16, DeviceVit, vit_init

    B = VIT_MB
    x, y = synthetic_images(2 * B * n, seed=0, hw=224, classes=1000)
    init = vit_init(VIT_B16, seed=0)
    perms = [np.random.default_rng([0, t]).permutation(len(x))[:n * B] for t in range(1, warmup + steps + 2)]
    res = {}
    for name in ("cdp-v2", "dp"):
        rule = None if name == "dp" else rule_by_name(name, n)
        torch.cuda.synchronize()
        free0 = torch.cuda.mem_get_info()[0]
        tr = DeviceVit.single_gpu(VIT_B16, B, n, rule, RN_MOMENTUM, inputs=x, labels=y, probe=True)
        torch.cuda.synchronize()
        alloc = free0 - torch.cuda.mem_get_info()[0]
        tr.set_params(init, -1)
        for t in range(warmup):
            tr.step(perms[t], RN_LR)
        tr.sync()
        with ClockSampler(0) as clk:
            for k in range(steps):
                tr.flush_l2()
                tr.mark(2 * k)
                tr.step(perms[warmup + k], RN_LR)
                tr.mark(2 * k + 1)
            tr.sync()
        ms = float(np.mean([tr.elapsed(2 * k, 2 * k + 1) for k in range(steps)]))
        losses, flags = tr.history(warmup + steps)
        assert np.all(np.isfinite(losses)) and not flags.any(), "non-finite ViT step"
        st = tr.stats()
        plan_peak = tr.plan.peak_bytes(st["record_bytes"])
        assert st["live_record_high_water_bytes"] == plan_peak, (st, plan_peak)
        r = {"value": round(n * B / (ms / 1e3), 1), "unit": UNIT, "ms_per_step": round(ms, 3),
             "peak_activation_bytes": st["live_record_high_water_bytes"],
             "activation_record_pool_bytes": st["activation_bytes"], "record_slots": st["record_slots"],
             "record_bytes": st["record_bytes"], "trainer_device_bytes_allocated": int(alloc),
             "gpu_launches": st["kernels_per_step"] * steps, "clocks": clk.summary(),
             "tensor_tflops_per_s": round(st["tensor_flops_per_step"] / (ms / 1e3) / 1e12, 1)}
        if profile and name == "cdp-v2":
            ops = tr.profile_step(perms[warmup + steps], RN_LR, serial=True)
            agg = kernel_table(ops)
            tot = sum(a[1] for a in agg.values())
            gemm = {k: a for k, a in agg.items() if a[2] > 0}
            dom = max(gemm, key=lambda k: gemm[k][1])
            d = gemm[dom]
            peak, src = peak_tensor()
            achieved = d[2] / (d[1] / 1e3) / 1e12
            r["roofline"] = {"bound": "tensor", "kernel": f"{dom} ({d[0]} launches)", "achieved": round(achieved, 1),
                             "peak": peak, "peak_source": src, "unit": "TFLOP/s", "frac": round(achieved / peak, 4),
                             "share_of_serial_step": round(d[1] / tot, 3)}
            r["kernel_breakdown"] = {
                k: {"launches": a[0], "ms": round(a[1], 3), "share": round(a[1] / tot, 3),
                    **({"tflops": round(a[2] / (a[1] / 1e3) / 1e12, 1)} if a[2] else
                       {"gbs": round(a[3] / (a[1] / 1e3) / 1e9, 1)})}
                for k, a in sorted(agg.items(), key=lambda kv: -kv[1][1])[:16]}
        tr.close()
        res[name] = r
    c, d = res["cdp-v2"], res["dp"]
    return {"workload": f"configs[3]: ViT-B/16 224x224, {n} sequential micro-batches of {B} on one GPU "
                        f"({n} stages, block-aligned), cdp-v2 vs dp, bf16 operands, fp32 master / momentum",
            "value": c["value"], "unit": UNIT, "ms_per_step": c["ms_per_step"], "cdp_v2": c, "dp": d,
            "peak_activation_cdp_over_dp": round(c["peak_activation_bytes"] / d["peak_activation_bytes"], 4),
            "expected_ratio_ref_costs_py": round((n + 1) / (2 * n), 4),
            "allocated_cdp_over_dp": round(c["trainer_device_bytes_allocated"] / d["trainer_device_bytes_allocated"], 4)}


def cpu_resnet_reference(model, ws, rule, sample_images, steps, threads):
    """The oracle port (oracle/resnet_torch.py, float64 torch-CPU autograd under the reference's `_advance`
    semantics) on `sample_images` images per micro-batch, one micro-batch per worker, `steps` steps."""
    import torch

    from oracle.resnet_torch import run_cdp
    from paper_2403_08837_b200.resnet import init_params, layer_specs, stage_partition, synthetic_images

    torch.set_num_threads(threads)
    if model == "vit_b16":
        from oracle.vit_torch import run_cdp as vit_cdp
        from paper_2403_08837_b200.vit import VIT_B16, stage_partition as vit_stages, vit_init, vit_units

        x, y = synthetic_images(sample_images * ws, seed=0, hw=224, classes=1000)
        fresh = None
        if rule is not None:
            stage = vit_stages(vit_units(**VIT_B16), ws)
            fresh = [[rule.reads_fresh(i, int(s)) for s in stage] for i in range(1, ws + 1)]
        init = vit_init(VIT_B16, 0)
        perms = [np.random.default_rng([0, t]).permutation(len(x)) for t in range(1, steps + 2)]
        vit_cdp(VIT_B16, init, x.astype(np.float64), y, ws, sample_images, perms[:1], RN_LR, RN_MOMENTUM, fresh)
        t0 = time.perf_counter()
        vit_cdp(VIT_B16, init, x.astype(np.float64), y, ws, sample_images, perms[1:steps + 1], RN_LR, RN_MOMENTUM,
                fresh)
        dt = (time.perf_counter() - t0) / steps
        return ws * sample_images / dt, dt * 1e3
    cfg, hw, classes = resnet_cfg(model)
    specs = layer_specs(cfg["widths"], cfg["depths"], 3, hw, cfg["block"], cfg["stem"], classes)
    x, y = synthetic_images(sample_images * ws, seed=0, hw=hw, classes=classes)
    fresh = None
    if rule is not None:
        stage = stage_partition(specs, ws)
        fresh = [[rule.reads_fresh(i, int(s)) for s in stage] for i in range(1, ws + 1)]
    init = init_params(specs, 0)
    perms = [np.random.default_rng([0, t]).permutation(len(x)) for t in range(1, steps + 2)]
    run_cdp(cfg["widths"], cfg["depths"], init, x.astype(np.float64), y, ws, sample_images, perms[:1], RN_LR,
            RN_MOMENTUM, fresh, block=cfg["block"], stem=cfg["stem"], classes=classes)  # warm-up
    t0 = time.perf_counter()
    run_cdp(cfg["widths"], cfg["depths"], init, x.astype(np.float64), y, ws, sample_images, perms[1:steps + 1],
            RN_LR, RN_MOMENTUM, fresh, block=cfg["block"], stem=cfg["stem"], classes=classes)
    dt = (time.perf_counter() - t0) / steps
    return ws * sample_images / dt, dt * 1e3


def resnet_workload(model, ws, rule_name, dtype):
    mb = RN_MB
    if model == "resnet18":
        what = "ResNet-18 CIFAR variant (3x3 stem, no max pool), 32x32x3, 10 classes"
    elif model == "vit_b16":
        what = "ViT-B/16 (torchvision layout), 224x224x3, 1000 classes, fp32 residual stream"
        mb = VIT_MB
        if dtype == "fp32":
            dtype = "fp32 (3xTF32, unfused attention: the parity mode)"
    else:
        what = "ResNet-50 (torchvision v1.5 layout), 224x224x3, 1000 classes"
    return (f"{what}; {rule_name}; one micro-batch of {mb} per GPU; {ws} stage(s) = {ws} GPU(s); {dtype} "
            f"operands, fp32 master/momentum; SGD lr {RN_LR} momentum {RN_MOMENTUM}")


def main_resnet(args, ws, rank, local):
    from paper_2403_08837_b200.dist import resolve

    model = args.model
    res = run_resnet(args, ws, rank, local, model, args.steps, args.warmup)
    # ---- comparison points at the same N (configs[2]: CDP-v2 vs the DP all-reduce baseline; configs[4]:
    # ZeRO-CDP P2P state passing vs the ZeRO-DP broadcast baseline).  Run on every rank; a failure of a
    # baseline is reported, not fatal to the headline.
    baselines = None
    if ws > 1 and not args.no_extras and args.rule == "cdp-v2" and not args.zero and model != "vit_b16":
        baselines = {}
        steps_v = max(3, min(args.steps, 20))
        for mode in ("dp-allreduce", "zero-cdp", "zero-dp"):
            try:
                baselines[mode] = run_resnet_variant(args, ws, rank, local, model, steps_v, 3, mode)
            except Exception as e:  # noqa: BLE001 - reported in the JSON line
                baselines[mode] = {"error": f"{type(e).__name__}: {e}"[:300]}
    if rank != 0:
        return None
    peak_note = ("configs[1]" if model == "resnet18" else
                 "configs[3]'s model, one micro-batch per GPU (N GPUs = N stages)" if model == "vit_b16" else
                 "configs[2] (north-star target; N GPUs = N stages)")
    out = {
        "metric": METRIC, "value": res["value"], "unit": UNIT, "n_gpus": ws, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": res["ms_per_step"], "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": args.dtype,
        "data": "synthetic (x ~ N(0,1) NHWC, uniform labels; numpy PCG64), deterministic He-normal init",
        "config": {"workload": resnet_workload(model, ws, args.rule, args.dtype), "baseline_config": peak_note,
                   "global_batch": ws * RN_MB, "micro_batch": RN_MB, "stages": ws, "rule": args.rule,
                   "parallelism": (f"dp{ws} (NCCL all-reduce of the flat gradient + update kernel)"
                                   if args.rule == "dp-allreduce" else
                                   f"{'zero-' if args.zero and ws > 1 else ''}cdp{ws} (one process per GPU, P2P "
                                   f"gradient hop ring, fused update on rank {ws - 1}"
                                   f"{', ZeRO-CDP P2P state passing' if args.zero and ws > 1 else ''})"),
                   "l2": "flushed (256 MiB memset) before every timed step"},
        "e2e": res["e2e"], "gpu_launches": res["gpu_launches"], "roofline": res["roofline"],
        "activation_bytes": res["activation_bytes"], "tensor_tflops_per_s": res["tensor_tflops_per_s"],
        "clocks": res["clocks"], "kernel_breakdown": res["kernel_breakdown"],
        "serial_step_ms": res["serial_step_ms"], "losses_first_last": res["losses_first_last"],
        "exposed_comm": res.get("exposed_comm"), "p2p": res.get("p2p"),
    }
    if args.zero and ws > 1:
        out["zero_cdp"] = {"state_bytes_received_per_step_rank0": res["zero_state_bytes_per_step"],
                           "what": "both theta version slots + momentum of every received tensor use (P2P copy "
                                   "kernels, ref comm.py:93-144 holder chain)",
                           "param_state_bytes_rank0": res["param_state_bytes"],
                           "layout": "two stage frames per rank (parameter-balanced, block-aligned stages); "
                                     "theta slots + momentum + compute copies + the gradient partial sum"}
    if baselines is not None:
        b = out["baselines"] = baselines
        if "value" in b.get("dp-allreduce", {}):
            b["cdp_over_dp_allreduce"] = round(out["value"] / b["dp-allreduce"]["value"], 4)
        if "value" in b.get("zero-cdp", {}) and "value" in b.get("zero-dp", {}):
            b["zero_cdp_over_zero_dp"] = round(b["zero-cdp"]["value"] / b["zero-dp"]["value"], 4)
        b["model_state_volume_per_device_ref_costs_py"] = {
            "zero_cdp": f"2(N-1)/N Psi_P = {2 * (ws - 1) / ws:.3f} Psi_P", "zero_dp": "2 Psi_P (ref costs.py:140-153)"}
    return out


def single_gpu_config1(dtype):
    """configs[0] on one GPU: 4 micro-batches x 32, 4 stages, CDP-v1 (+ activation bytes vs DP)."""
    from paper_2403_08837_b200.device import DeviceMlpTrainer
    from paper_2403_08837_b200.executor import plan_live_peak
    from paper_2403_08837_b200.rules import rule_by_name
    from paper_2403_08837_b200.training import make_mlp_task

    task = make_mlp_task(**CONFIG1)
    res = {}
    for rname in ("cdp-v1", "dp"):
        rule = None if rname == "dp" else rule_by_name(rname, 4)
        tr = DeviceMlpTrainer(task.model.dims, 32, 4, 1, rule, dtype=dtype, momentum=MOMENTUM, inputs=task.inputs,
                              targets=task.targets)
        tr.set_params(np.concatenate(task.init_params()), which=-1)
        for t in range(1, 11):
            tr.step(task.permutation(t), LR)
        ms = []
        for k in range(100):
            tr.flush_l2()
            tr.mark(0)
            tr.step(task.permutation(11 + k), LR)
            tr.mark(1)
            ms.append(tr.elapsed(0, 1))
        live = plan_live_peak(tr.plan, task.model.dims, 32, 2 if dtype == "bf16" else 8) if tr.plan is not None else {}
        res[rname] = (float(np.mean(ms)), tr.stats()["activation_bytes"], live.get("peak_live_records"))
        tr.close()
    sps, cms, kind = cpu_reference(task, [[False] * 4 for _ in range(4)], 8, 1, 1)
    return {"workload": "configs[0]: 3072-256-256-256-10, 4 micro-batches x 32 on 1 GPU (4 worker streams), cdp-v1",
            "value": round(128 / (res["cdp-v1"][0] / 1e3), 1), "unit": UNIT, "ms_per_step": round(res["cdp-v1"][0], 5),
            "dp_value": round(128 / (res["dp"][0] / 1e3), 1),
            "activation_bytes": {"cdp": res["cdp-v1"][1], "dp": res["dp"][1],
                                 "ratio": round(res["cdp-v1"][1] / res["dp"][1], 4),
                                 "note": "allocated record slots = the peak of live record bytes over the "
                                         "executed op order; layer 1's 3072-wide records dominate and are live "
                                         "for all 4 micro-batches in both schedules"},
            "live_records_peak": {"cdp": res["cdp-v1"][2], "dp": res["dp"][2],
                                  "ratio": (round(res["cdp-v1"][2] / res["dp"][2], 4)
                                            if res["cdp-v1"][2] and res["dp"][2] else None),
                                  "ref": "(N+1)/2 vs N records per micro-batch, ref costs.py:111-115"},
            "cpu_baseline": {"value": round(sps, 2), "unit": UNIT, "cores": 1, "kind": kind,
                             "sample": "8 steps after 1 warm-up, reference Cython kernel, fp64, single thread"}}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=100)
    ap.add_argument("--warmup", type=int, default=10)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--dtype", default="bf16", choices=["bf16", "fp32"])
    ap.add_argument("--rule", default="cdp-v2", choices=["cdp-v2", "cdp-v1", "dp", "dp-allreduce"])
    ap.add_argument("--model", default="resnet50", choices=["resnet18", "resnet50", "vit_b16", "mlp"])
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-extras", action="store_true", help="skip the resnet50 / config-1 sub-lines at N=1")
    ap.add_argument("--zero", action="store_true", help="ZeRO-CDP state passing (ResNets, N > 1)")
    args = ap.parse_args()
    ws, rank, local = dist_env()

    if args.model != "mlp":
        if args.zero and args.rule != "cdp-v2":
            raise SystemExit("--zero uses the CDP-v2 placement (ref schedule.py:471)")
        if args.impl == "reference":
            if rank != 0:
                return
            from paper_2403_08837_b200.dist import resolve

            threads = os.cpu_count() or 1
            n = max(1, min(args.steps, 2))
            sample = 16 if args.model == "resnet18" else 1 if args.model == "vit_b16" else 2
            sps, ms = cpu_resnet_reference(args.model, ws, None if args.rule == "dp-allreduce" else resolve(args.rule, ws),
                                           sample, n, threads)
            desc = (f"{n} steps (after 1 warm-up) of the {ws}-micro-batch CDP step on {sample} images per "
                    f"micro-batch (of {VIT_MB if args.model == 'vit_b16' else RN_MB}), float64 torch-CPU oracle port, "
                    f"{threads} threads")
            print(json.dumps({
                "impl": "reference", "metric": METRIC, "value": round(sps, 3), "unit": UNIT, "n_gpus": ws,
                "steps": n, "warmup": 1, "ms_per_step": round(ms, 3), "higher_is_better": True, "scaling": "weak",
                "vs_baseline": None, "dtype": "f64", "data": "synthetic",
                "config": {"workload": resnet_workload(args.model, ws, args.rule, "fp64")},
                "cpu_baseline": {"value": round(sps, 3), "unit": UNIT, "cores": threads, "kind": "port",
                                 "sample": desc, "host_cpus": os.cpu_count()},
                "e2e": {"value": round(sps, 3), "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
            }), flush=True)
            return
        if ws > 1:
            import torch

            torch.cuda.set_device(local % torch.cuda.device_count())
            torch.distributed.init_process_group("nccl" if torch.cuda.device_count() >= ws else "gloo")
        out = main_resnet(args, ws, rank, local)
        if rank == 0:
            if ws == 1 and not args.no_extras:
                if args.model in ("resnet18", "resnet50"):
                    other = "resnet18" if args.model == "resnet50" else "resnet50"
                    r = run_resnet(args, 1, 0, local, other, 20, 5, e2e=True)
                    out[other] = {"workload": resnet_workload(other, 1, args.rule, args.dtype),
                                  "baseline_config": "configs[1]" if other == "resnet18" else "configs[2]",
                                  "value": r["value"], "unit": UNIT, "ms_per_step": r["ms_per_step"],
                                  "e2e": r["e2e"], "tensor_tflops_per_s": r["tensor_tflops_per_s"],
                                  "roofline": r["roofline"], "activation_bytes": r["activation_bytes"],
                                  "clocks": r["clocks"], "kernel_breakdown": r["kernel_breakdown"]}
                out["vit_b16_single_gpu_cdp"] = vit_single_gpu(4, 5, 3, profile=True)
                v12 = vit_single_gpu(12, 3, 2)
                out["vit_b16_single_gpu_cdp_n12"] = {k: v12[k] for k in (
                    "workload", "value", "unit", "ms_per_step", "peak_activation_cdp_over_dp",
                    "expected_ratio_ref_costs_py", "allocated_cdp_over_dp")}
                out["vit_b16_single_gpu_cdp_n12"]["peak_activation_bytes"] = {
                    "cdp_v2": v12["cdp_v2"]["peak_activation_bytes"], "dp": v12["dp"]["peak_activation_bytes"]}
                out["single_gpu_cdp"] = single_gpu_config1(args.dtype)
            if ws == 1 and not args.no_cpu_baseline:
                threads = os.cpu_count() or 1
                from paper_2403_08837_b200.dist import resolve

                sample = 16 if args.model == "resnet18" else 1 if args.model == "vit_b16" else 2
                sps, _ms = cpu_resnet_reference(args.model, 1, resolve(args.rule, 1), sample, 2, threads)
                out["cpu_baseline"] = {"value": round(sps, 3), "unit": UNIT, "cores": threads, "kind": "port",
                                       "sample": f"2 steps (after 1 warm-up) of the same CDP step on {sample} "
                                                 f"images (of {VIT_MB if args.model == 'vit_b16' else RN_MB}), "
                                                 f"float64 torch-CPU oracle port, {threads} threads",
                                       "host_cpus": os.cpu_count()}
            print(json.dumps(out), flush=True)
        if ws > 1:
            import torch

            torch.distributed.barrier()
            torch.distributed.destroy_process_group()
        return

    if args.impl == "reference":
        if rank != 0:
            return
        from paper_2403_08837_b200.dist import resolve
        from paper_2403_08837_b200.executor import layer_stages

        task = make_deep_task(ws)
        fresh = expanded_fresh(None if args.rule == "dp-allreduce" else resolve(args.rule, ws), ws,
                               layer_stages(len(DEEP_DIMS) - 1, ws))
        cores = min(ws, os.cpu_count() or 1)
        n = max(1, min(args.steps, 5))
        sps, ms, kind = cpu_reference(task, fresh, n, 1, cores)
        desc = (f"{n} full steps (after 1 warm-up) of the {ws}-micro-batch step, fp64, reference Cython kernel, "
                f"{'one process per micro-batch' if cores > 1 else 'single thread'}")
        print(json.dumps({
            "impl": "reference", "metric": METRIC, "value": round(sps, 3), "unit": UNIT, "n_gpus": ws, "steps": n,
            "warmup": 1, "ms_per_step": round(ms, 3), "higher_is_better": True, "scaling": "weak",
            "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": {"workload": workload_name(ws, args.rule, "fp64")},
            "cpu_baseline": {"value": round(sps, 3), "unit": UNIT, "cores": cores, "kind": kind, "sample": desc,
                             "host_cpus": os.cpu_count()},
            "e2e": {"value": round(sps, 3), "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
        }), flush=True)
        return

    if ws > 1:
        import torch

        torch.cuda.set_device(local)
        torch.distributed.init_process_group("nccl")
    out, task, rule, ls = run_ours(args, ws, rank, local)
    if rank == 0:
        if not args.no_cpu_baseline and ws == 1:
            sps, _ms, kind = cpu_reference(task, expanded_fresh(rule, ws, ls), 4, 1, 1)
            out["cpu_baseline"] = {"value": round(sps, 3), "unit": UNIT, "cores": 1, "kind": kind,
                                   "sample": "4 steps (after 1 warm-up) of the same 1-micro-batch step (B=128, 8 "
                                             "layers), fp64, reference Cython kernel, single thread",
                                   "host_cpus": os.cpu_count()}
            out["single_gpu_cdp"] = single_gpu_config1(args.dtype)
        print(json.dumps(out), flush=True)
    if ws > 1:
        import torch

        torch.distributed.barrier()
        torch.distributed.destroy_process_group()


if __name__ == "__main__":
    main()
