#!/usr/bin/env python
"""CDP training-step benchmark on B200 (contract: DESIGN.md §Measurement).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
                    [--dtype bf16|fp32] [--rule cdp-v1|cdp-v2|dp]

Workload (round 1): BASELINE.json configs[0], the config the reference can
execute — the stage MLP 3072-256-256-256-10, N = 4 micro-batches = stages =
workers, B = 32, softmax-xent, SGD lr 0.05 momentum 0.9, CDP-v1 (the
reference's CPU path, timed beside it).  configs[1..4] (ResNet / ViT) are not
built yet.  One "step" = one training step over N*B = 128
samples, the whole CDP step on the device (forward, backward, gradient hops,
fused update) as one CUDA graph.

Prints ONE JSON line (rank 0).  `value` = samples/s of the device-timed step
(CUDA events on the trainer stream around each graph launch, inputs resident
in HBM, L2 flushed with a 256 MiB memset before every timed step, max over
ranks); `e2e` = the same through the public API with host (pinned) inputs
copied H2D inside each step and the step loss read back every step.
`--impl reference` times the reference's own CPU implementation of the step
(its compiled Cython kernel from oracle/_ref, the engine loop restated in
oracle/engine.py) on the host cores, one process per micro-batch.
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
    BASELINE = json.load(_fh)
METRIC = BASELINE["metric"]
UNIT = "samples/s"
CONFIG1 = dict(n=4, micro_batch_size=32, seed=0, width=256, in_dim=3072, out_dim=10, loss_kind="xent")
LR, MOMENTUM = 0.05, 0.9


def dist_env():
    ws = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return ws, rank, local


def workload_name(rule, dtype):
    return (f"config1 stage-MLP 3072-256-256-256-10, N=4 micro-batches/stages/workers, B=32, xent, "
            f"{rule}, {dtype}, SGD lr {LR} momentum {MOMENTUM}")


# ----------------------------------------------------------------------------- clocks
class ClockSampler:
    """nvml samples of SM clock and throttle reasons, ~1 kHz, during the timed region."""

    REASONS = {
        0x1: "gpu_idle", 0x2: "applications_clocks_setting", 0x4: "sw_power_cap", 0x8: "hw_slowdown",
        0x10: "sync_boost", 0x20: "sw_thermal_slowdown", 0x40: "hw_thermal_slowdown",
        0x80: "hw_power_brake_slowdown", 0x100: "display_clock_setting",
    }

    def __init__(self, index=0):
        self.samples, self.reasons, self.ok = [], set(), False
        try:
            import pynvml

            pynvml.nvmlInit()
            self.nv = pynvml
            self.h = pynvml.nvmlDeviceGetHandleByIndex(index)
            self.max_mhz = pynvml.nvmlDeviceGetMaxClockInfo(self.h, pynvml.NVML_CLOCK_SM)
            self.ok = True
        except Exception:
            self.max_mhz = None
        self._stop = threading.Event()

    def _run(self):
        while not self._stop.is_set():
            try:
                self.samples.append(self.nv.nvmlDeviceGetClockInfo(self.h, self.nv.NVML_CLOCK_SM))
                r = self.nv.nvmlDeviceGetCurrentClocksEventReasons(self.h)
                for bit, name in self.REASONS.items():
                    if r & bit and bit != 0x1:
                        self.reasons.add(name)
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
        return {"sm_mhz": statistics.median(self.samples) if self.samples else None,
                "sm_max_mhz": self.max_mhz, "reasons": sorted(self.reasons), "samples": len(self.samples)}


# ----------------------------------------------------------------------------- reference arm
def _ref_worker(args):
    dims, theta, x, labels = args
    from oracle import kernels as OK

    mod = OK.load_reference_kernels()
    return mod.mlp_value_grad(dims, theta, x, None, labels, 1)


def run_reference(steps, warmup, rule="cdp-v1", pool_size=None, sample_steps=None):
    """The reference's CPU step: its compiled Cython kernel per micro-batch, engine loop restated
    (ref engine.py:66-116).  Returns (samples/s, cores, kind, description)."""
    from oracle import engine as OE
    from oracle import kernels as OK

    mod = OK.load_reference_kernels()
    kind = "reference" if mod is not None else "port"
    task = OE.make_mlp_task(**CONFIG1)
    fresh = OE.fresh_table(rule, task.n)
    cur = task.init_params()
    prev = [p.copy() for p in cur]
    vel = [np.zeros_like(p) for p in cur]
    cores = pool_size or 1
    pool = None
    if cores > 1:
        import multiprocessing as mp

        pool = mp.get_context("fork").Pool(cores)

    def grads_fn_parallel(batches, params_per_mb):
        jobs = [(task.dims, np.concatenate(params_per_mb[i]), batches[i][0], batches[i][1].astype(np.int64))
                for i in range(task.n)]
        return pool.map(_ref_worker, jobs)

    def one_step(t):
        nonlocal cur, prev
        batches = task.micro_batches(t)
        if pool is None:
            kern = (lambda d, th, x, y, l, k: mod.mlp_value_grad(d, th, x, y, l, k)) if mod else OK.mlp_value_grad

            def gfn(params, x, y):
                loss, g = kern(task.dims, np.concatenate(params), x, None, y.astype(np.int64), 1)
                return loss, OE.split(g, task.stage_sizes)

            new, _ = OE.advance(task, cur, prev, t, batches, LR, fresh, MOMENTUM, vel, grads_fn=gfn)
        else:
            params = [[cur[j] if (fresh is None or fresh[i][j]) else prev[j] for j in range(task.n)]
                      for i in range(task.n)]
            res = grads_fn_parallel(batches, params)
            it = iter(res)

            def gfn(_params, _x, _y):
                loss, g = next(it)
                return loss, OE.split(g, task.stage_sizes)

            new, _ = OE.advance(task, cur, prev, t, batches, LR, fresh, MOMENTUM, vel, grads_fn=gfn)
        prev, cur = cur, new

    for t in range(1, warmup + 1):
        one_step(t)
    n = sample_steps or steps
    t0 = time.perf_counter()
    for t in range(warmup + 1, warmup + n + 1):
        one_step(t)
    dt = time.perf_counter() - t0
    if pool is not None:
        pool.close()
    sps = n * task.n * task.micro_batch_size / dt
    desc = (f"{n} steps of the config-1 {rule} step (N=4 x B=32, fp64, momentum {MOMENTUM}) after {warmup} warm-up; "
            f"{'reference Cython kernel (oracle/_ref)' if kind == 'reference' else 'C restatement (oracle)'}"
            f"{', one process per micro-batch' if pool is not None else ', single thread'}")
    return sps, cores, kind, desc, dt / n * 1e3


# ----------------------------------------------------------------------------- our arm
def run_ours(args, ws, rank, local):
    import torch

    torch.cuda.set_device(local)
    from paper_2403_08837_b200.device import DeviceMlpTrainer
    from paper_2403_08837_b200.rules import rule_by_name
    from paper_2403_08837_b200.training import make_mlp_task

    task = make_mlp_task(**CONFIG1)
    rule = None if args.rule == "dp" else rule_by_name(args.rule, task.n)
    tr = DeviceMlpTrainer(task.model.dims, task.micro_batch_size, task.n, 1, rule, dtype=args.dtype,
                          momentum=MOMENTUM, inputs=task.inputs, targets=task.targets)
    tr.set_params(np.concatenate(task.init_params()), which=-1)
    perms = [task.permutation(t) for t in range(1, args.warmup + args.steps + 2)]
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
    step_ms = [tr.elapsed(2 * k, 2 * k + 1) for k in range(K)]
    ms = float(np.mean(step_ms))
    if ws > 1:
        t = torch.tensor([ms], device="cuda")
        torch.distributed.all_reduce(t, op=torch.distributed.ReduceOp.MAX)
        ms = float(t.item())
    samples_per_step = task.n * task.micro_batch_size
    value = ws * samples_per_step / (ms / 1e3)
    losses, flags = tr.history()
    assert np.all(np.isfinite(losses)) and not flags.any(), "non-finite step in the timed region"
    stats = tr.stats()

    # ---- e2e: public API, pinned host inputs copied H2D each step, loss read back each step
    B = samples_per_step
    x_pin = torch.empty((B, task.model.dims[0]), dtype=torch.float32, pin_memory=True)
    y_pin = torch.empty((B,), dtype=torch.int32, pin_memory=True)
    h2d = x_pin.numel() * 4 + y_pin.numel() * 4 + 16 + B * 4  # batch + labels + control block + row table
    d2h = 8 + 12
    batches = []
    for k in range(K + 2):
        p = perms[k % len(perms)]
        batches.append((task.inputs[p].astype(np.float32), task.targets[p].astype(np.int32)))
    for k in range(2):  # warm the host path
        x_pin.numpy()[:] = batches[k][0]
        y_pin.numpy()[:] = batches[k][1]
        tr.step_host_batch_ptr(x_pin.data_ptr(), y_pin.data_ptr(), LR)
        tr.last()
    e2e_ms = []
    for k in range(K):
        x_pin.numpy()[:] = batches[k + 2][0]
        y_pin.numpy()[:] = batches[k + 2][1]
        tr.flush_l2()
        tr.mark(0)
        tr.step_host_batch_ptr(x_pin.data_ptr(), y_pin.data_ptr(), LR)
        loss, fl = tr.last()
        tr.mark(1)
        e2e_ms.append(tr.elapsed(0, 1))
    e2e = float(np.mean(e2e_ms))
    if ws > 1:
        t = torch.tensor([e2e], device="cuda")
        torch.distributed.all_reduce(t, op=torch.distributed.ReduceOp.MAX)
        e2e = float(t.item())

    # ---- roofline: the dominant kernel = stage-1 weight-grad GEMM fused with the mid ring hop
    op = tr.op_index(1, 2, 1)
    R = 20
    kms = []
    for _ in range(R):
        tr.flush_l2()
        kms.append(tr.time_op(op, 4, -1))
    k_ms = float(np.median(kms))
    d0, d1 = task.model.dims[0], task.model.dims[1]
    p1 = d0 * d1 + d1
    esz = 2 if args.dtype == "bf16" else 8  # bf16 operand, or fp32 hi+lo
    alg_bytes = p1 * 8 + task.micro_batch_size * (d0 + d1) * esz  # read S + write S, read H and dZ
    with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) if os.path.exists(
            os.path.join(ROOT, "MEASURED_PEAKS.json")) else open(os.devnull) as fh:
        try:
            peaks = json.load(fh)
            peak, peak_src = float(peaks["hbm_gbs"]), "measured"
        except Exception:
            peak, peak_src = 6650.0, "fallback"
    achieved = alg_bytes / (k_ms / 1e3) / 1e9
    traffic = None
    tp = os.path.join(ROOT, "profiles", "round1_wgrad_hop_traffic.json")
    if os.path.exists(tp):
        with open(tp) as fh:
            traffic = json.load(fh).get(args.dtype, {}).get("dram_bytes_per_launch")

    # ---- activation memory CDP vs DP (same model, same executor)
    other = DeviceMlpTrainer(task.model.dims, task.micro_batch_size, task.n, 1,
                             None if rule is not None else rule_by_name("cdp-v2", task.n), dtype=args.dtype)
    act_other = other.stats()["activation_bytes"]
    other.close()
    act_cdp, act_dp = (stats["activation_bytes"], act_other) if rule is not None else (act_other, stats["activation_bytes"])

    out = {
        "metric": METRIC, "value": round(value, 1), "unit": UNIT, "n_gpus": ws, "steps": K, "warmup": args.warmup,
        "ms_per_step": round(ms, 5), "higher_is_better": True, "scaling": "weak", "vs_baseline": None,
        "dtype": args.dtype, "data": "synthetic (reference make_mlp_task seed 0, numpy PCG64)",
        "config": {"workload": workload_name(args.rule, args.dtype), "global_batch": ws * samples_per_step,
                   "micro_batch": task.micro_batch_size, "n_micro_batches": task.n, "rule": args.rule,
                   "parallelism": f"single-GPU CDP x{ws} replicas" if ws > 1 else "single-GPU CDP (4 worker streams)",
                   "l2": "flushed (256 MiB memset) before every timed step; working set < L2"},
        "e2e": {"value": round(ws * samples_per_step / (e2e / 1e3), 1), "unit": UNIT, "h2d_bytes_per_step": h2d,
                "d2h_bytes_per_step": d2h, "ms_per_step": round(e2e, 5)},
        "gpu_launches": stats["kernels_per_step"] * K,
        "roofline": {"bound": "hbm", "kernel": "stage-1 wgrad GEMM + fused mid ring hop (gemm_tc_kernel<EpiWgrad>)",
                     "achieved": round(achieved, 1), "peak": peak, "peak_source": peak_src, "unit": "GB/s",
                     "frac": round(achieved / peak, 4), "traffic": traffic,
                     "algorithmic_bytes_per_launch": alg_bytes, "launch_us": round(k_ms * 1e3, 2)},
        "activation_bytes": {"cdp": act_cdp, "dp": act_dp, "ratio": round(act_cdp / act_dp, 4)},
        "clocks": clk.summary(),
    }
    return out, tr


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=200)
    ap.add_argument("--warmup", type=int, default=10)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--dtype", default="bf16", choices=["bf16", "fp32"])
    ap.add_argument("--rule", default="cdp-v1", choices=["cdp-v1", "cdp-v2", "dp"])
    ap.add_argument("--no-cpu-baseline", action="store_true")
    args = ap.parse_args()
    ws, rank, local = dist_env()

    if args.impl == "reference":
        if rank != 0:
            return
        cores = min(4, os.cpu_count() or 1)
        n = max(1, min(args.steps, 60))
        sps, cores, kind, desc, ms = run_reference(n, min(args.warmup, 3), rule=args.rule, pool_size=cores)
        print(json.dumps({
            "impl": "reference", "metric": METRIC, "value": round(sps, 3), "unit": UNIT, "n_gpus": ws, "steps": n,
            "warmup": min(args.warmup, 3), "ms_per_step": round(ms, 3), "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": {"workload": workload_name(args.rule, "fp64")},
            "cpu_baseline": {"value": round(sps, 3), "unit": UNIT, "cores": cores, "kind": kind, "sample": desc,
                             "host_cpus": os.cpu_count()},
            "e2e": {"value": round(sps, 3), "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
        }), flush=True)
        return

    if ws > 1:
        import torch

        torch.distributed.init_process_group("nccl")
    out, tr = run_ours(args, ws, rank, local)
    if rank == 0:
        if not args.no_cpu_baseline and ws == 1:
            sps, cores, kind, desc, _ = run_reference(12, 1, rule=args.rule, pool_size=None)
            out["cpu_baseline"] = {"value": round(sps, 3), "unit": UNIT, "cores": cores, "kind": kind,
                                   "sample": desc, "host_cpus": os.cpu_count()}
        print(json.dumps(out), flush=True)
    tr.close()
    if ws > 1:
        import torch

        torch.distributed.destroy_process_group()


if __name__ == "__main__":
    main()
