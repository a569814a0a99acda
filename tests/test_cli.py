"""CLI (ref cli.py): config errors and plan subcommands on CPU; train-toy / trace on the GPU."""

import json
import os

import pytest

from paper_2403_08837_b200.cli import EXIT_CONFIG, EXIT_OK, main


def test_simulate_writes_reference_timeline_text(tmp_path):
    assert main(["simulate", "--scheme", "multi-gpu-cdp", "--n", "4", "--out", str(tmp_path)]) == EXIT_OK
    text = (tmp_path / "timeline.txt").read_text()
    assert text.startswith("# cyclicdp-timeline v1\n# scheme=multi-gpu-cdp n=4")
    assert sum(1 for l in text.splitlines() if l.startswith("task\t")) == 2 * 16 * 4
    assert sum(1 for l in text.splitlines() if l.startswith("comm\t")) == 16 * 4


def test_timeline_text_matches_reference_format_exactly(tmp_path):
    """Byte-for-byte: one golden plan re-rendered the reference's way."""
    import gzip

    from conftest import GOLDEN
    from paper_2403_08837_b200 import ParallelismConfig, Scheme, make_homogeneous_profile
    from paper_2403_08837_b200.comm import scheduled_timeline
    from paper_2403_08837_b200.export import timeline_to_text

    cases = {c["name"]: c for c in json.load(gzip.open(os.path.join(GOLDEN, "plans.json.gz"), "rt"))}
    case = cases["sched-multi-gpu-cdp-cdp-v2-n3-s2"]
    tl = scheduled_timeline(ParallelismConfig(Scheme.MULTI_GPU_CDP, 3, 2, 2), make_homogeneous_profile(3, 36, 180, 0),
                            "cdp-v2")
    lines = timeline_to_text(tl).splitlines()
    tasks = [l.split("\t") for l in lines if l.startswith("task")]
    assert [[t[1], int(t[2]), int(t[3]), t[4], int(t[5]), int(t[6]), int(t[7]), int(t[8])] for t in tasks] == \
        [[c[5], c[6], c[7], c[0], c[1], c[2], c[3], c[4]] for c in case["tasks"]]


def test_validate_and_config_errors(tmp_path, capsys):
    assert main(["validate", "--scheme", "single-gpu-cdp", "--n", "3"]) == EXIT_OK
    assert main(["validate", "--scheme", "pp", "--n", "3"]) == EXIT_CONFIG
    cfg = tmp_path / "c.json"
    cfg.write_text(json.dumps({"task": "resnet"}))
    assert main(["train-toy", "--config", str(cfg), "--out", str(tmp_path)]) == EXIT_CONFIG
    cfg.write_text("{not json")
    assert main(["train-toy", "--config", str(cfg), "--out", str(tmp_path)]) == EXIT_CONFIG


@pytest.mark.gpu
def test_train_toy_on_gpu_matches_reference_trajectories(cuda, tmp_path):
    from oracle import engine as OE

    assert main(["train-toy", "--task", "mlp", "--n", "4", "--batch", "4", "--steps", "10", "--lr", "0.05",
                 "--out", str(tmp_path)]) == EXIT_OK
    rows = (tmp_path / "trajectories.csv").read_text().splitlines()
    assert rows[0] == "# cyclicdp-trajectories-csv v1" and rows[1] == "step,rule,loss"
    summary = json.loads((tmp_path / "summary.json").read_text())
    ref = OE.run_experiment(OE.make_mlp_task(4, 4, 0), steps=10, lr=0.05)
    for rule, run in ref.items():
        assert abs(summary["final_losses"][rule] - run.losses[-1]) <= 1e-5 * abs(run.losses[-1])


@pytest.mark.gpu
def test_trace_executed_schedule_respects_plan(cuda, tmp_path):
    assert main(["trace", "--n", "4", "--rule", "cdp-v2", "--out", str(tmp_path)]) == EXIT_OK
    text = (tmp_path / "executed.txt").read_text()
    assert text.startswith("# cyclicdp-timeline v1")
    assert sum(1 for l in text.splitlines() if l.startswith("exec\t")) == 2 * 16 * 3
