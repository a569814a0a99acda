"""Command line (ref `cli.py:1-381`, the hot-path subset).

    python -m paper_2403_08837_b200 train-toy [--config cfg.json | flags] [--dtype fp32|bf16] --out DIR
    python -m paper_2403_08837_b200 simulate --scheme S --n N [--rule R] --out DIR     (timeline text)
    python -m paper_2403_08837_b200 validate --scheme S --n N [--rule R]
    python -m paper_2403_08837_b200 trace --n N [--rule R] --out DIR                   (executed schedule)

`train-toy` keeps the reference's JSON keys (`task, n, micro_batch_size,
steps, lr, seed, rules, momentum`, ref `cli.py:186-195`), flags, artefacts
(`trajectories.csv` in `cyclicdp-trajectories-csv v1`, `summary.json` with
the same keys) and exit codes (0 ok, 2 config error, 3 validation failure,
5 divergence); the step runs on the B200 (`dtype`, `weight_decay` are
additions).  `trace` runs a few CDP steps of the MLP on the GPU with
device-clock stamps around every task and writes the executed schedule in
`cyclicdp-timeline v1` (+ `exec` lines), then checks that the executed order
respects every dependency of the planned timeline (forward sweep, backward
sweep, forward-before-backward, ring-hop order).
"""

from __future__ import annotations

import argparse
import json
import sys
from pathlib import Path

EXIT_OK, EXIT_CONFIG, EXIT_VALIDATION, EXIT_MISMATCH, EXIT_DIVERGENCE = 0, 2, 3, 4, 5


class CliError(Exception):
    pass


def _write(out: Path, name: str, text: str) -> None:
    out.mkdir(parents=True, exist_ok=True)
    (out / name).write_text(text)


def _train_toy_config(args):
    if args.config:
        doc = json.loads(Path(args.config).read_text())
        cfg = dict(task=doc.get("task", "quadratic"), n=int(doc.get("n", 4)), batch=int(doc.get("micro_batch_size", 2)),
                   steps=int(doc.get("steps", 200)), lr=float(doc.get("lr", 0.1)), seed=int(doc.get("seed", 0)),
                   rules=tuple(doc.get("rules", ["dp", "cdp-v1", "cdp-v2"])), momentum=float(doc.get("momentum", 0.0)),
                   dtype=str(doc.get("dtype", args.dtype)), weight_decay=float(doc.get("weight_decay", args.weight_decay)))
    else:
        cfg = dict(task=args.task, n=args.n, batch=args.batch, steps=args.steps, lr=args.lr, seed=args.seed,
                   rules=tuple(r.strip() for r in args.rules.split(",") if r.strip()), momentum=args.momentum,
                   dtype=args.dtype, weight_decay=args.weight_decay)
    if cfg["task"] not in ("quadratic", "quad", "mlp"):
        raise CliError(f"unknown task {cfg['task']!r}")
    if cfg["dtype"] not in ("fp32", "bf16"):
        raise CliError(f"unknown dtype {cfg['dtype']!r}")
    if cfg["n"] < 1 or cfg["batch"] < 1 or cfg["steps"] < 1:
        raise CliError("n, micro_batch_size and steps must be >= 1")
    return cfg


def cmd_train_toy(args) -> int:
    try:
        cfg = _train_toy_config(args)
    except (CliError, ValueError, OSError, json.JSONDecodeError) as exc:
        print(f"config error: {exc}", file=sys.stderr)
        return EXIT_CONFIG
    from .export import trajectories_to_csv
    from .training import make_mlp_task, make_quadratic_task, run_experiment

    task = (make_mlp_task(cfg["n"], cfg["batch"], cfg["seed"]) if cfg["task"] == "mlp"
            else make_quadratic_task(cfg["n"], cfg["batch"], cfg["seed"]))
    try:
        result = run_experiment(task, cfg["rules"], steps=cfg["steps"], lr=cfg["lr"], momentum=cfg["momentum"],
                                dtype=cfg["dtype"], weight_decay=cfg["weight_decay"])
    except ValueError as exc:
        print(f"config error: {exc}", file=sys.stderr)
        return EXIT_CONFIG
    out = Path(args.out)
    _write(out, "trajectories.csv", trajectories_to_csv(result))
    summary = {
        "task": cfg["task"], "n": cfg["n"], "micro_batch_size": cfg["batch"], "steps": cfg["steps"], "lr": cfg["lr"],
        "seed": cfg["seed"], "momentum": cfg["momentum"], "final_losses": result.final_losses(),
        "max_pairwise_trajectory_divergence": result.max_pairwise_divergence(),
        "diverged": {name: run.diverged_at for name, run in result.runs.items()},
        "dtype": cfg["dtype"], "weight_decay": cfg["weight_decay"], "device": "B200 (sm_100a)",
    }
    _write(out, "summary.json", json.dumps(summary, indent=2, sort_keys=True) + "\n")
    diverged = {k: v for k, v in summary["diverged"].items() if v is not None}
    if diverged:
        for name, step in diverged.items():
            print(f"divergence: rule {name} at step {step}", file=sys.stderr)
        return EXIT_DIVERGENCE
    for name, loss in result.final_losses().items():
        print(f"{name:>8} final loss {loss:.6e}")
    return EXIT_OK


def _build(args):
    from .comm import scheduled_timeline
    from .profiles import CostWeights, ParallelismConfig, Scheme, make_homogeneous_profile

    try:
        scheme = Scheme(args.scheme)
        cfg = ParallelismConfig(scheme, args.n, args.batch, args.training_steps,
                                CostWeights(getattr(args, "forward_cost", 1), getattr(args, "backward_cost", 1)))
        prof = make_homogeneous_profile(args.n, args.total_params, args.total_acts, args.boundary_acts)
        return scheduled_timeline(cfg, prof, args.rule)
    except NotImplementedError as exc:
        raise CliError(str(exc))


def cmd_simulate(args) -> int:
    from .export import timeline_to_text
    from .schedule import validate_timeline

    try:
        tl = _build(args)
    except (CliError, ValueError) as exc:
        print(f"config error: {exc}", file=sys.stderr)
        return EXIT_CONFIG
    rep = validate_timeline(tl)
    _write(Path(args.out), "timeline.txt", timeline_to_text(tl))
    for v in rep.violations:
        print(f"violation[{v.kind}]: {v.message}", file=sys.stderr)
    return EXIT_OK if rep.ok else EXIT_VALIDATION


def cmd_validate(args) -> int:
    from .schedule import validate_timeline

    try:
        tl = _build(args)
    except (CliError, ValueError) as exc:
        print(f"config error: {exc}", file=sys.stderr)
        return EXIT_CONFIG
    rep = validate_timeline(tl)
    if rep.ok:
        print(f"ok: {len(tl.tasks)} tasks, {len(tl.comm_events)} comm events")
        return EXIT_OK
    for v in rep.violations:
        print(f"violation[{v.kind}]: {v.message}", file=sys.stderr)
    return EXIT_VALIDATION


def executed_order_violations(tl, executed: dict) -> list:
    """Dependencies of the planned timeline that the executed stamps break."""
    from .schedule import TaskKind

    n = tl.n
    bad = []
    for (kind, i, j, t), (s, e) in executed.items():
        if kind is TaskKind.FORWARD and j > 1:
            p = executed.get((TaskKind.FORWARD, i, j - 1, t))
            if p and p[1] > s:
                bad.append(f"forward ({i},{j},{t}) started before stage {j - 1} finished")
        if kind is TaskKind.BACKWARD:
            f = executed.get((TaskKind.FORWARD, i, j, t))
            if f and f[1] > s:
                bad.append(f"backward ({i},{j},{t}) started before its forward finished")
            if j < n:
                nx = executed.get((TaskKind.BACKWARD, i, j + 1, t))
                if nx and nx[0] > s:
                    bad.append(f"backward ({i},{j},{t}) started before backward of stage {j + 1}")
            if i > 1:
                prev = executed.get((TaskKind.BACKWARD, i - 1, j, t))
                if prev and prev[1] > e:
                    bad.append(f"hop ({i},{j},{t}) finished before the previous worker's hop")
    return bad


def _planned_peak(tl, record_bytes) -> int:
    """The plan's peak live record bytes (records live from F.start through B.end, ref costs.py:157-170)."""
    from .costs import activation_records

    delta = [0] * (tl.horizon + 2)
    for _dev, lo, hi, stage, _i, _t in activation_records(tl):
        delta[max(1, lo)] += int(record_bytes[stage - 1])
        delta[min(tl.horizon, hi) + 1] -= int(record_bytes[stage - 1])
    acc, peak = 0, 0
    for g in range(1, tl.horizon + 1):
        acc += delta[g]
        peak = max(peak, acc)
    return peak


def cmd_trace(args) -> int:
    import numpy as np

    from .device import DeviceMlpTrainer
    from .export import executed_to_text
    from .profiles import ParallelismConfig, Scheme
    from .rules import rule_by_name
    from .schedule import build_cdp_timeline, build_dp_timeline
    from .training import make_mlp_task

    n = args.n
    task = make_mlp_task(n=n, micro_batch_size=args.batch, seed=0, width=args.width, in_dim=args.width,
                         out_dim=10, loss_kind="xent")
    rule = None if args.rule == "dp" else rule_by_name(args.rule, n)
    tr = DeviceMlpTrainer(task.model.dims, args.batch, n, 1, rule, dtype=args.dtype, inputs=task.inputs,
                          targets=task.targets)
    tr.set_params(np.concatenate(task.init_params()), which=-1)
    executed = {}
    for t in range(1, args.training_steps + 1):
        executed.update(tr.trace_step(task.permutation(t), 0.05, t))
    tr.close()
    cfg = ParallelismConfig(Scheme.SINGLE_GPU_DP if rule is None else Scheme.SINGLE_GPU_CDP, n, args.batch,
                            args.training_steps)
    tl = build_dp_timeline(cfg) if rule is None else build_cdp_timeline(cfg, rule)
    _write(Path(args.out), "executed.txt", executed_to_text(tl, executed))
    if args.training_steps >= 3:
        import json

        from .accounting import executed_activation, executed_balance
        from .costs import activation_records

        esz = 2 if args.dtype == "bf16" else 8
        rb = [args.batch * ((d + 15) // 16 * 16) * esz for d in task.model.dims[:-1]]  # executor.record_bytes
        act = executed_activation(executed, rb, args.training_steps)
        planned = _planned_peak(tl, rb)
        bal = executed_balance(tl, executed)
        rep = {"executed": {"peak_activation_bytes": act.peak_bytes, "steady_max_bytes": act.steady_max_bytes,
                            "steady_min_bytes": act.steady_min_bytes, "steady_mean_bytes": round(act.mean_bytes, 1)},
               "planned_peak_activation_bytes": planned, "balance": bal}
        _write(Path(args.out), "accounting.json", json.dumps(rep, indent=1))
        print(f"executed peak activation {act.peak_bytes} B (planned {planned} B); "
              f"max hops per worker per boundary {bal['max_sends_or_receives_per_worker']}")
    bad = executed_order_violations(tl, executed)
    for b in bad:
        print(f"violation[executed-order]: {b}", file=sys.stderr)
    print(f"{len(executed)} tasks executed; {len(bad)} ordering violations")
    return EXIT_OK if not bad else EXIT_VALIDATION


def _profile_args(p):
    p.add_argument("--total-params", type=int, default=480)
    p.add_argument("--total-acts", type=int, default=4800)
    p.add_argument("--boundary-acts", type=int, default=240)


def build_parser() -> argparse.ArgumentParser:
    from .profiles import Scheme

    parser = argparse.ArgumentParser(prog="paper_2403_08837_b200", description="B200-native cyclic data parallelism")
    sub = parser.add_subparsers(dest="command", required=True)

    p = sub.add_parser("train-toy", help="run the update rules on a toy task (on the GPU)")
    p.add_argument("--config")
    p.add_argument("--task", default="quadratic", choices=["quadratic", "quad", "mlp"])
    p.add_argument("--n", type=int, default=4)
    p.add_argument("--batch", type=int, default=2)
    p.add_argument("--steps", type=int, default=200)
    p.add_argument("--lr", type=float, default=0.1)
    p.add_argument("--seed", type=int, default=0)
    p.add_argument("--momentum", type=float, default=0.0)
    p.add_argument("--rules", default="dp,cdp-v1,cdp-v2")
    p.add_argument("--dtype", default="fp32", choices=["fp32", "bf16"])
    p.add_argument("--weight-decay", type=float, default=0.0)
    p.add_argument("--out", default="out")
    p.set_defaults(func=cmd_train_toy)

    for name, fn in (("simulate", cmd_simulate), ("validate", cmd_validate)):
        p = sub.add_parser(name)
        p.add_argument("--scheme", required=True, choices=[s.value for s in Scheme])
        p.add_argument("--n", type=int, required=True)
        p.add_argument("--batch", type=int, default=1)
        p.add_argument("--training-steps", type=int, default=4)
        p.add_argument("--rule", default="cdp-v2")
        p.add_argument("--forward-cost", type=int, default=1)
        p.add_argument("--backward-cost", type=int, default=1)
        _profile_args(p)
        if name == "simulate":
            p.add_argument("--out", default="out")
        p.set_defaults(func=fn)

    p = sub.add_parser("trace", help="run CDP steps on the GPU and export the executed schedule")
    p.add_argument("--n", type=int, default=4)
    p.add_argument("--batch", type=int, default=16)
    p.add_argument("--width", type=int, default=64)
    p.add_argument("--training-steps", type=int, default=3)
    p.add_argument("--rule", default="cdp-v2")
    p.add_argument("--dtype", default="bf16", choices=["fp32", "bf16"])
    p.add_argument("--out", default="out")
    p.set_defaults(func=cmd_trace)
    return parser


def main(argv=None) -> int:
    args = build_parser().parse_args(argv)
    return args.func(args)


if __name__ == "__main__":
    sys.exit(main())
