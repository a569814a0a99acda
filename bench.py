#!/usr/bin/env python
"""CDP training-step benchmark on B200 (contract: DESIGN.md §Measurement).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
                    [--dtype bf16|fp32] [--rule cdp-v2|cdp-v1|dp]
    torchrun --nproc-per-node N bench.py --gpus N ...

Workload (round 1; ResNet / ViT layer kernels are not built yet, DESIGN.md
§Scope): BASELINE configs[1]'s structure — CDP-v2, ONE micro-batch per GPU,
N = micro-batches = stages = GPUs — on the stage MLP family of configs[0]:
an 8-layer tanh MLP 3072-256x7-10 (softmax-xent, SGD lr 0.05 momentum 0.9),
micro-batch B = 128 per GPU, the 8 layers grouped into N contiguous stages.
Per-GPU work is the same at every N (weak scaling).  One step = one training
step of the whole job: every rank's forward + backward, the per-layer
gradient hops rank -> rank+1 over peer memory, the fused update on the last
rank, the parameter pulls — one CUDA graph per rank, no collective.

At N = 1 the line also carries `single_gpu_cdp`: configs[0] itself (4-layer
3072-256-256-256-10, 4 micro-batches of 32 on one GPU, CDP-v1), the
reference's own CPU-runnable case, with its CPU time beside it.

`value` = samples/s of the device-timed step (CUDA events on each rank's
trainer stream around each graph launch, inputs resident in HBM, L2 flushed
by a 256 MiB memset before every timed step, max over ranks); `e2e` = the
same through the public API from pinned host inputs copied H2D inside every
step with the step loss read back every step.  `--impl reference` times the
reference's own CPU implementation (its compiled Cython kernel, oracle/_ref,
under the restated engine loop) with one process per micro-batch.
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


def single_gpu_config1(dtype):
    """configs[0] on one GPU: 4 micro-batches x 32, 4 stages, CDP-v1 (+ activation bytes vs DP)."""
    from paper_2403_08837_b200.device import DeviceMlpTrainer
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
        res[rname] = (float(np.mean(ms)), tr.stats()["activation_bytes"])
        tr.close()
    sps, cms, kind = cpu_reference(task, [[False] * 4 for _ in range(4)], 8, 1, 1)
    return {"workload": "configs[0]: 3072-256-256-256-10, 4 micro-batches x 32 on 1 GPU (4 worker streams), cdp-v1",
            "value": round(128 / (res["cdp-v1"][0] / 1e3), 1), "unit": UNIT, "ms_per_step": round(res["cdp-v1"][0], 5),
            "dp_value": round(128 / (res["dp"][0] / 1e3), 1),
            "activation_bytes": {"cdp": res["cdp-v1"][1], "dp": res["dp"][1],
                                 "ratio": round(res["cdp-v1"][1] / res["dp"][1], 4)},
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
    ap.add_argument("--no-cpu-baseline", action="store_true")
    args = ap.parse_args()
    ws, rank, local = dist_env()

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
