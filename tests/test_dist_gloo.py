"""Host side of multi-GPU CDP on CPU: world_size-2 gloo process group.

Covers the IPC-handle exchange (the only thing torch.distributed does for
the CDP step), rank plan compilation on every rank, and that the rank plans
of a job form exactly one gradient chain per layer (first ... last) with
pulls on every rank but the updater.
"""

import os
import socket

import numpy as np
import pytest
import torch.distributed as dist
import torch.multiprocessing as mp


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_2403_08837_b200.dist import exchange_handles
        from paper_2403_08837_b200.executor import compile_rank_plan, layer_stages
        from paper_2403_08837_b200.rules import min_delay_rule

        mine = bytes([rank + 1]) * 64
        got = exchange_handles(mine)
        ops = compile_rank_plan(world, rank, min_delay_rule(world), layer_stages(4, world))
        q.put((rank, [h[0] for h in got], ops.tolist()))
        bad = None
        try:
            exchange_handles(b"short" if rank == 0 else bytes(64))
        except ValueError as e:
            bad = str(e)
        q.put((rank, "bad", bad))
    finally:
        dist.destroy_process_group()


def test_gloo_world2_handle_exchange_and_rank_plans():
    world = 2
    port = _free_port()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    out = [q.get(timeout=120) for _ in range(2 * world)]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    plans = {}
    for item in out:
        if item[1] == "bad":
            assert item[2] is not None  # every rank rejects a malformed peer handle
            continue
        rank, first_bytes, ops = item
        assert first_bytes == [1, 2]
        plans[rank] = np.array(ops)
    # rank 0 = worker 1 (first hop, pulls), rank 1 = worker 2 (last hop = updater, no pulls)
    assert set(plans[0][plans[0][:, 0] == 1][:, 6]) == {0}
    assert set(plans[1][plans[1][:, 0] == 1][:, 6]) == {2}
    assert (plans[0][:, 0] == 2).sum() == 4 and (plans[1][:, 0] == 2).sum() == 0
