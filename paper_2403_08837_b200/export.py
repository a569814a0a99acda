"""Stable text / CSV formats shared with the reference (ref `export.py:17-202`).

* `timeline_to_text`     — `cyclicdp-timeline v1` (ref `export.py:45-81`), the
                           planned schedule, byte-identical to the reference's
                           for the same Timeline;
* `trajectories_to_csv`  — `cyclicdp-trajectories-csv v1` (ref `export.py:194-202`);
* `executed_to_text`     — the schedule the GPU actually ran (trace mode of the
                           trainer): the same task records in the same format,
                           followed by `exec` lines with the measured start/end
                           of every task (ns on the device clock), so the
                           executed order can be diffed against the plan.
"""

from __future__ import annotations

import csv
import io
from fractions import Fraction

from .schedule import Timeline

TIMELINE_FORMAT = "cyclicdp-timeline v1"
TRAJECTORY_FORMAT = "cyclicdp-trajectories-csv v1"


def _fmt(v) -> str:
    if isinstance(v, Fraction):
        return str(v)
    if isinstance(v, float):
        return repr(v)
    return str(v)


def timeline_to_text(tl: Timeline) -> str:
    """task <device> <start> <duration> <kind> <mb> <stage> <step> <version>
    comm <boundary> <kind> <src> <dst> <stage> <mb|-> <payload> <depth>"""
    out = [f"# {TIMELINE_FORMAT}", f"# scheme={tl.scheme.value} n={tl.n} horizon={tl.horizon} devices={len(tl.devices)}"]
    out += ["\t".join(map(str, ("task", t.device, t.start, t.duration, t.kind.value, t.micro_batch, t.stage,
                                 t.training_step, t.param_version))) for t in tl.tasks]
    out += ["\t".join(map(str, ("comm", e.boundary, e.kind.value, e.src, e.dst, e.stage,
                                 "-" if e.micro_batch is None else e.micro_batch, _fmt(e.payload), e.depth)))
            for e in tl.comm_events]
    return "\n".join(out) + "\n"


def trajectories_to_csv(result) -> str:
    buf = io.StringIO()
    buf.write(f"# {TRAJECTORY_FORMAT}\n")
    w = csv.writer(buf)
    w.writerow(["step", "rule", "loss"])
    for name, run in result.runs.items():
        for step, loss in enumerate(run.losses, start=1):
            w.writerow([step, name, repr(float(loss))])
    return buf.getvalue()


def executed_to_text(tl: Timeline, executed: dict) -> str:
    """Planned records plus `exec <device> <kind> <mb> <stage> <step> <start_ns> <end_ns>` lines.

    `executed` maps (kind, micro_batch, stage, step) -> (start_ns, end_ns) as
    returned by `DeviceMlpTrainer.trace_step`."""
    lines = timeline_to_text(tl).rstrip("\n").split("\n")
    lines.append("# executed: device-clock ns of each task's first kernel start and last kernel end")
    index = tl.task_index()
    for key in sorted(executed, key=lambda k: (executed[k][0], str(k))):
        t = index.get(key)
        dev = t.device if t is not None else "?"
        s, e = executed[key]
        lines.append("\t".join(map(str, ("exec", dev, key[0].value, key[1], key[2], key[3], s, e))))
    return "\n".join(lines) + "\n"
