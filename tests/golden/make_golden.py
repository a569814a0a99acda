"""Generate the golden fixtures from the reference itself.

Run in the build container (needs /root/reference):

    python tests/golden/make_golden.py

It imports the UNMODIFIED reference package from a temporary copy of
/root/reference/pkg (the tree is read-only; the Cython kernel is built in
the copy with the reference's own setup.py) and records:

* plans.json.gz   task lists, comm events, validator / reduction / balance
                  results and measured peak activations for DP, CDP (v1, v2,
                  generic) and ZeRO plans over N, steps, cost weights;
* kernels.npz     mlp_value_grad / quad_value_grad outputs on seeded inputs;
* toy_runs.npz    run_experiment losses, final params and version traces on
                  small MLP (mse, xent) and quadratic tasks, momentum 0 / 0.9;
* closed_form.json  closed_form_costs (ref costs.py:64-153) activation per device and state
                  volume per step for the hot-path schemes over n, micro-batch and profiles;
* config1.npz     config-1 shape (3072-256-256-256-10, N=4, B=32, xent):
                  data checksums, 20-step losses and a fixed sample of the
                  final parameters for dp / cdp-v1 / cdp-v2, momentum 0.9.

Nothing under /root/reference is read at test time; the tests only read
these files.
"""

from __future__ import annotations

import gzip
import json
import os
import shutil
import subprocess
import sys
import tempfile

import numpy as np

OUT = os.path.dirname(os.path.abspath(__file__))


def load_reference():
    tmp = tempfile.mkdtemp(prefix="cdp_ref_")
    shutil.copytree("/root/reference/pkg", os.path.join(tmp, "pkg"))
    subprocess.check_call([sys.executable, "setup.py", "build_ext", "--inplace"], cwd=os.path.join(tmp, "pkg"),
                          stdout=subprocess.DEVNULL, stderr=subprocess.DEVNULL)
    sys.path.insert(0, os.path.join(tmp, "pkg", "src"))
    import cyclicdp  # noqa: F401
    from cyclicdp.training import BACKEND_NAME

    assert BACKEND_NAME == "compiled", BACKEND_NAME
    return tmp


def enc_task(t):
    return [t.kind.value, t.micro_batch, t.stage, t.training_step, t.param_version, t.device, t.start, t.duration]


def enc_event(e):
    return [e.boundary, e.kind.value, e.src, e.dst, str(e.payload), e.stage, e.micro_batch, e.participants, e.depth]


def plans():
    from cyclicdp import (ParallelismConfig, Scheme, build_cdp_timeline, build_dp_timeline, generic_rule,
                          make_homogeneous_profile, validate_timeline)
    from cyclicdp.comm import balance_report, scheduled_timeline, verify_gradient_reduction
    from cyclicdp.costs import measure_costs
    from cyclicdp.profiles import CostWeights
    from cyclicdp.schedule import build_zero_timeline

    cases = []

    def record(name, tl, profile=None):
        rep = validate_timeline(tl)
        entry = {
            "name": name,
            "horizon": tl.horizon,
            "devices": [[d.id, d.gpu, d.capacity, d.param_model.value, list(d.owned_stages)] for d in tl.devices],
            "tasks": [enc_task(t) for t in tl.tasks],
            "events": [enc_event(e) for e in tl.comm_events],
            "violations": [[v.kind, v.message] for v in rep.violations],
            "steady": list(tl.steady_window()),
        }
        if tl.comm_events:
            entry["reduction"] = [[c.stage, c.training_step, c.complete_at, c.first_fresh_read, c.ok]
                                  for c in verify_gradient_reduction(tl)]
            br = balance_report(tl)
            entry["balance"] = [br.max_sends, br.min_sends, str(br.mean_sends), list(br.deep_boundaries),
                                list(br.cyclic_depth_flags)]
        if profile is not None and tl.cfg.training_steps >= 3:
            entry["peak_activation"] = str(measure_costs(tl, profile).peak_activation_memory_per_device)
        cases.append(entry)

    for n in (1, 2, 3, 4, 5, 8):
        for steps in (2, 3):
            for w in ((1, 1), (1, 2), (2, 3)):
                cw = CostWeights(*w)
                prof = make_homogeneous_profile(n, 12 * n, 60 * n, 0)
                for sch in (Scheme.SINGLE_GPU_DP, Scheme.MULTI_GPU_DP):
                    cfg = ParallelismConfig(sch, n, 2, steps, cw)
                    record(f"{sch.value}-n{n}-s{steps}-w{w[0]}{w[1]}", build_dp_timeline(cfg), prof)
                    if w == (1, 1):
                        record(f"sched-{sch.value}-n{n}-s{steps}", scheduled_timeline(cfg, prof), prof)
                for sch in (Scheme.SINGLE_GPU_CDP, Scheme.MULTI_GPU_CDP):
                    for rule in ("cdp-v1", "cdp-v2"):
                        cfg = ParallelismConfig(sch, n, 2, steps, cw)
                        try:
                            tl = build_cdp_timeline(cfg, rule)
                        except Exception as exc:  # infeasible combos are recorded too
                            cases.append({"name": f"{sch.value}-{rule}-n{n}-s{steps}-w{w[0]}{w[1]}",
                                          "error": type(exc).__name__})
                            continue
                        record(f"{sch.value}-{rule}-n{n}-s{steps}-w{w[0]}{w[1]}", tl, prof)
                        if w == (1, 1):
                            record(f"sched-{sch.value}-{rule}-n{n}-s{steps}", scheduled_timeline(cfg, prof, rule), prof)
                if w == (1, 1):
                    for sch in (Scheme.ZERO_DP, Scheme.ZERO_CDP):
                        cfg = ParallelismConfig(sch, n, 2, steps, cw)
                        record(f"zero-{sch.value}-n{n}-s{steps}", build_zero_timeline(cfg, prof, sch is Scheme.ZERO_CDP), prof)
                        record(f"sched-{sch.value}-n{n}-s{steps}", scheduled_timeline(cfg, prof), prof)
    # a feasible generic rule and heterogeneous payloads
    from cyclicdp import ModelProfile

    table = [[False, False, True], [False, True, True], [False, False, False]]
    cfg = ParallelismConfig(Scheme.MULTI_GPU_CDP, 3, 2, 3)
    hp = ModelProfile((5, 7, 11), (30, 20, 10), 12)
    record("generic-n3", build_cdp_timeline(cfg, generic_rule(table)), hp)
    record("sched-generic-n3", scheduled_timeline(cfg, hp, generic_rule(table)), hp)
    with gzip.open(os.path.join(OUT, "plans.json.gz"), "wt") as fh:
        json.dump(cases, fh, separators=(",", ":"))
    return len(cases)


def kernels():
    from cyclicdp.training import kernels as K

    rng = np.random.default_rng(1234)
    out = {}
    k = 0
    for dims in ((4, 6, 6, 2), (7, 5, 3), (12, 9, 9, 9, 4), (3072, 16, 10)):
        for kind in (0, 1):
            b = 5 if dims[0] < 100 else 3
            p = sum(dims[j] * dims[j + 1] + dims[j + 1] for j in range(len(dims) - 1))
            theta = rng.normal(0, 0.5, size=p)
            x = rng.normal(size=(b, dims[0]))
            y = rng.normal(size=(b, dims[-1])) if kind == 0 else None
            lab = rng.integers(0, dims[-1], size=b).astype(np.int64) if kind == 1 else None
            loss, g = K.mlp_value_grad(dims, theta, x, y, lab, kind)
            out[f"mlp{k}_dims"] = np.array(dims)
            out[f"mlp{k}_kind"] = np.array(kind)
            out[f"mlp{k}_theta"] = theta
            out[f"mlp{k}_x"] = x
            out[f"mlp{k}_y"] = y if y is not None else np.zeros((0,))
            out[f"mlp{k}_labels"] = lab if lab is not None else np.zeros((0,), dtype=np.int64)
            out[f"mlp{k}_loss"] = np.array(loss)
            out[f"mlp{k}_grad"] = g
            k += 1
    out["n_mlp"] = np.array(k)
    a = rng.normal(size=(9, 9))
    th = rng.normal(size=9)
    tg = rng.normal(size=(4, 9))
    loss, g = K.quad_value_grad(a, th, tg)
    out.update(quad_a=a, quad_theta=th, quad_targets=tg, quad_loss=np.array(loss), quad_grad=g)
    np.savez_compressed(os.path.join(OUT, "kernels.npz"), **out)


def toy_runs():
    from cyclicdp.training import make_mlp_task, make_quadratic_task, run_experiment

    out = {}
    specs = {
        "mlp_mse": lambda: make_mlp_task(n=4, micro_batch_size=4, seed=3, width=8, in_dim=6, out_dim=3, loss_kind="mse"),
        "mlp_xent": lambda: make_mlp_task(n=4, micro_batch_size=4, seed=5, width=8, in_dim=6, out_dim=3, loss_kind="xent"),
        "mlp_xent_n3": lambda: make_mlp_task(n=3, micro_batch_size=6, seed=7, width=10, in_dim=5, out_dim=4, loss_kind="xent"),
        "quad": lambda: make_quadratic_task(n=4, micro_batch_size=2, seed=11),
    }
    for name, mk in specs.items():
        task = mk()
        out[f"{name}_inputs"] = task.inputs
        out[f"{name}_targets"] = task.targets
        out[f"{name}_init"] = np.concatenate(task.init_params())
        out[f"{name}_perm3"] = np.concatenate([np.concatenate([b[0].ravel()]) for b in task.micro_batches(3)])
        for mom in (0.0, 0.9):
            res = run_experiment(task, steps=20, lr=0.05, momentum=mom, record_trace=True)
            for rule, run in res.runs.items():
                key = f"{name}_m{int(mom * 10)}_{rule}"
                out[key + "_losses"] = np.array(run.losses)
                out[key + "_final"] = np.concatenate(run.final_params)
                out[key + "_trace"] = np.array(run.trace, dtype=np.int64)
                out[key + "_diverged"] = np.array(-1 if run.diverged_at is None else run.diverged_at)
    np.savez_compressed(os.path.join(OUT, "toy_runs.npz"), **out)


CONFIG1 = dict(n=4, micro_batch_size=32, seed=0, width=256, in_dim=3072, out_dim=10, loss_kind="xent")


def config1(steps=20):
    from cyclicdp.training import make_mlp_task, run_experiment

    task = make_mlp_task(**CONFIG1)
    out = {
        "inputs_sum": np.array(task.inputs.sum()),
        "inputs_sample": task.inputs.ravel()[::997].copy(),
        "targets": task.targets,
        "perm_step": np.concatenate([task.micro_batches(t)[0][0][:, 0] for t in (1, 2, 7)]),
    }
    total = sum(task.model.stage_sizes)
    sample = np.random.default_rng(99).choice(total, size=4096, replace=False)
    sample.sort()
    out["sample_idx"] = sample
    out["init_sample"] = np.concatenate(task.init_params())[sample]
    for mom in (0.0, 0.9):
        res = run_experiment(task, steps=steps, lr=0.05, momentum=mom)
        for rule, run in res.runs.items():
            flat = np.concatenate(run.final_params)
            key = f"m{int(mom * 10)}_{rule}"
            out[key + "_losses"] = np.array(run.losses)
            out[key + "_sample"] = flat[sample]
            out[key + "_stage_sq"] = np.array([float(np.dot(p, p)) for p in run.final_params])
    np.savez_compressed(os.path.join(OUT, "config1.npz"), **out)


def closed_forms():
    from cyclicdp import ParallelismConfig, Scheme, make_homogeneous_profile
    from cyclicdp.costs import closed_form_costs

    out = []
    for sch in (Scheme.SINGLE_GPU_DP, Scheme.SINGLE_GPU_CDP, Scheme.MULTI_GPU_DP, Scheme.MULTI_GPU_CDP,
                Scheme.ZERO_DP, Scheme.ZERO_CDP):
        for n in (1, 2, 3, 4, 8):
            for b in (1, 2, 5):
                for pp, pa in ((12, 60), (7, 3), (480, 4800)):
                    prof = make_homogeneous_profile(n, pp * n, pa * n, 1)
                    r = closed_form_costs(ParallelismConfig(sch, n, b, 3), prof)
                    out.append([sch.value, n, b, pp * n, pa * n, str(r.peak_activation_memory_per_device),
                                str(r.state_comm_volume_per_training_step)])
    with open(os.path.join(OUT, "closed_form.json"), "w") as fh:
        json.dump(out, fh)
    return len(out)


if __name__ == "__main__":
    tmp = load_reference()
    try:
        print("plans:", plans())
        print("closed forms:", closed_forms())
        kernels()
        toy_runs()
        if "--skip-config1" not in sys.argv:
            config1()
    finally:
        shutil.rmtree(tmp, ignore_errors=True)
    print("golden fixtures written to", OUT)
