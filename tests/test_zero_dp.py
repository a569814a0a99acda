"""ZeRO-DP baseline (ref comm.py:108-124: the owner of each stage broadcasts it, gradients reduce to
the owner, which alone updates it; `paper_2403_08837_b200.resnet.ZeroDpRank`).

CPU: the host protocol over a world-size-2 gloo group with a host-memory stand-in trainer (stage
ranges, broadcast / reduce order, owner-only update, repack of the non-owned tensors) reproduces
the DP update.  GPU: two processes on one GPU (gloo) running the real trainer are bit-identical to
the DP all-reduce baseline run in one process.
"""

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


class _HostTrainer:
    """Stand-in for DeviceResNet(dp_allreduce=True): 4 tensors in 2 stages, theta slots on the host,
    gradient g = (rank + 1) * theta_cur (deterministic), SGD without momentum."""

    dp_allreduce = True

    def __init__(self, rank):
        self.rank = rank
        self.specs = [None] * 4
        self.stage = np.array([1, 1, 2, 2], dtype=np.int32)
        self.base = np.array([0, 3, 5, 9])
        self.P = 12
        self.t = 1
        self.theta = [torch.arange(12, dtype=torch.float32) + 1.0, torch.arange(12, dtype=torch.float32) + 1.0]
        self.g = torch.zeros(12)
        self.packed = []

    def tensor_bases(self):
        return self.base

    def stream_handle(self):
        return 0

    def partial_tensor(self):
        return self.g

    def theta_tensor(self, which=0):
        return self.theta[self.t & 1 if which == 0 else (self.t & 1) ^ 1]

    def pack_range(self, which, t0, t1):
        self.packed.append((self.t, t0, t1))

    def step(self, perm, lr):
        self.g.copy_(self.theta[self.t & 1] * (self.rank + 1))
        self.lr = lr
        self.t += 1

    def apply_update(self, t0, t1):
        p = (self.t - 1) & 1
        lo, hi = int(self.base[t0]), int(self.base[t1]) if t1 < 4 else self.P
        self.theta[p ^ 1][lo:hi] = self.theta[p][lo:hi] - self.lr / 2 * self.g[lo:hi]


def _host_worker(rank, world, port, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_2403_08837_b200.resnet import ZeroDpRank

        tr = _HostTrainer(rank)
        zd = ZeroDpRank(tr)
        for _ in range(3):
            zd.step(None, 0.1)
        zd.broadcast()
        q.put((rank, zd.ranges, zd.bytes_per_step, tr.theta_tensor(0).numpy().copy(), tr.packed))
    finally:
        dist.destroy_process_group()


def test_zero_dp_host_protocol_gloo_world2():
    world, port = 2, _free_port()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_host_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    out = sorted([q.get(timeout=120) for _ in range(world)], key=lambda o: o[0])
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    # DP reference: g_sum = (1 + 2) * theta, theta' = theta - lr / N * g_sum
    th = np.arange(12, dtype=np.float32) + 1.0
    for _ in range(3):
        th = th - np.float32(0.1 / 2) * (th * np.float32(3.0))
    for rank, ranges, nbytes, theta, packed in out:
        assert ranges == [(0, 2, 0, 5), (2, 4, 5, 12)]
        assert nbytes == 8 * (7 if rank == 0 else 5)
        np.testing.assert_allclose(theta, th, rtol=1e-6)
        other = (2, 4) if rank == 0 else (0, 2)
        assert [(t0, t1) for _, t0, t1 in packed] == [other] * 4  # one repack per broadcast


def _gpu_worker(rank, world, port, q, steps):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from oracle.resnet_torch import init_flat
        from paper_2403_08837_b200.resnet import DeviceResNet, ZeroDpRank, synthetic_cifar

        W, D, MB = (64, 128), (1, 1), 8
        x, y = synthetic_cifar(world * MB * 2, 0, hw=16, classes=10)
        init = init_flat(W, D, seed=0)
        perms = [np.random.default_rng([9, t]).permutation(len(x))[: world * MB] for t in range(1, steps + 1)]
        tr = DeviceResNet(W, D, MB, world, rank, None, "fp32", 0.9, inputs=x, labels=y, image_hw=16,
                          dp_allreduce=True)
        tr.set_params(init, -1)
        tr.connect([tr.region()] * world)
        zd = ZeroDpRank(tr)
        for k in range(steps):
            zd.step(perms[k][rank * MB:(rank + 1) * MB], 0.05)
        zd.broadcast()
        tr.sync()
        q.put((rank, tr.get_params(0)))
        tr.close()
    finally:
        dist.destroy_process_group()


@pytest.mark.gpu
def test_zero_dp_two_processes_match_dp_allreduce(cuda):
    world, steps, port = 2, 3, _free_port()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_gpu_worker, args=(r, world, port, q, steps)) for r in range(world)]
    for p in procs:
        p.start()
    out = sorted([q.get(timeout=600) for _ in range(world)], key=lambda o: o[0])
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    # the DP all-reduce baseline in one process (tests/test_gpu_resnet.py's construction)
    from oracle.resnet_torch import init_flat
    from paper_2403_08837_b200.resnet import DeviceResNet, synthetic_cifar

    W, D, MB = (64, 128), (1, 1), 8
    x, y = synthetic_cifar(world * MB * 2, 0, hw=16, classes=10)
    init = init_flat(W, D, seed=0)
    perms = [np.random.default_rng([9, t]).permutation(len(x))[: world * MB] for t in range(1, steps + 1)]
    tr = [DeviceResNet(W, D, MB, world, r, None, "fp32", 0.9, inputs=x, labels=y, image_hw=16, dp_allreduce=True)
          for r in range(world)]
    regions = [t.region() for t in tr]
    for t in tr:
        t.set_params(init, -1)
        t.connect(regions)
    for k in range(steps):
        for r, t in enumerate(tr):
            t.step(perms[k][r * MB:(r + 1) * MB], 0.05)
        for t in tr:
            t.sync()
        g = [t.partial_tensor() for t in tr]
        total = g[0] + g[1]
        for gi in g:
            gi.copy_(total)
        torch.cuda.synchronize()
        for t in tr:
            t.apply_update()
    for t in tr:
        t.sync()
    want = tr[0].get_params(0)
    for t in tr:
        t.close()
    for rank, params in out:
        assert np.array_equal(params, want), (rank, float(np.abs(params - want).max()))
