"""Multi-GPU CDP over torch.distributed: one process per GPU (rank r = worker r+1).

torch.distributed is plumbing only: it exchanges the 64-byte CUDA IPC handles
of every rank's shared region once (`exchange_handles`) and, for reporting,
reduces per-rank losses.  The training step itself never calls a collective:
gradients hop rank -> rank+1 inside the fused weight-gradient kernels over
peer memory and parameters are pulled from the updater (see
`csrc/mlp_kernels.cuh`, `RingFlags`).

`CdpRankGroup` wires one rank; `run_experiment_dist` is the distributed
counterpart of `training.run_experiment` for a single rule (each rank runs
its micro-batch; the losses are the mean over ranks; final parameters come
from the updater rank, which holds every stage's newest version).
"""

from __future__ import annotations

import numpy as np

from .device import DeviceMlpTrainer
from .executor import layer_stages
from .rules import UpdateRule, rule_by_name


def exchange_handles(local: bytes, group=None) -> list:
    """all_gather of each rank's IPC handle (works with gloo or nccl)."""
    import torch.distributed as dist

    out = [None] * dist.get_world_size(group)
    dist.all_gather_object(out, local, group=group)
    for h in out:
        if not isinstance(h, (bytes, bytearray)) or len(h) != 64:
            raise ValueError("malformed IPC handle from a peer rank")
    return [bytes(h) for h in out]


def resolve(rule, n):
    if rule is None or rule == "dp":
        return None
    return rule if isinstance(rule, UpdateRule) else rule_by_name(rule, n)


class CdpRankGroup:
    """This process's rank of a multi-GPU CDP job over an MLP with layers grouped into world stages."""

    def __init__(self, dims, micro_batch: int, loss_kind: int, rule, dtype: str = "bf16", momentum: float = 0.0,
                 weight_decay: float = 0.0, inputs=None, targets=None, group=None):
        import torch.distributed as dist

        self.rank = dist.get_rank(group)
        self.world = dist.get_world_size(group)
        n_layers = len(dims) - 1
        self.layer_stage = layer_stages(n_layers, self.world)
        self.trainer = DeviceMlpTrainer.for_rank(dims, micro_batch, self.world, self.rank, loss_kind,
                                                 resolve(rule, self.world), dtype=dtype, momentum=momentum,
                                                 weight_decay=weight_decay, inputs=inputs, targets=targets,
                                                 layer_stage=self.layer_stage)
        self.group = group
        self.micro_batch = micro_batch

    def connect(self, init_params: np.ndarray):
        self.trainer.set_params(init_params, which=-1)
        self.trainer.connect_ipc(exchange_handles(self.trainer.ipc_handle(), self.group))

    def step(self, perm_global: np.ndarray, lr: float):
        """perm_global: world*B rows; this rank trains on its micro-batch (rows rank*B..)."""
        b = self.micro_batch
        self.trainer.step(perm_global[self.rank * b:(self.rank + 1) * b], lr)

    def losses(self, steps: int) -> np.ndarray:
        import torch
        import torch.distributed as dist

        local, _flags = self.trainer.history(steps)
        t = torch.tensor(local, dtype=torch.float64, device="cuda")
        dist.all_reduce(t, group=self.group)
        return (t / self.world).cpu().numpy()

    def close(self):
        self.trainer.close()


def run_experiment_dist(task, rule="cdp-v2", steps: int = 10, lr=0.05, momentum: float = 0.0, dtype: str = "bf16"):
    """One rule on world ranks; task.n must equal the world size (one micro-batch per GPU)."""
    import torch.distributed as dist

    world = dist.get_world_size()
    if task.n != world:
        raise ValueError("run_experiment_dist needs task.n == world size")
    lr_of = lr if callable(lr) else (lambda t: lr)
    g = CdpRankGroup(task.model.dims, task.micro_batch_size, task.model.loss_code, rule, dtype=dtype,
                     momentum=momentum, inputs=task.inputs, targets=task.targets)
    g.connect(np.concatenate(task.init_params()))
    for t in range(1, steps + 1):
        g.step(task.permutation(t), lr_of(t))
    g.trainer.sync()
    if g.trainer.ring_error():
        raise RuntimeError(f"rank {g.rank}: cross-GPU ring protocol timed out")
    losses = g.losses(steps)
    final = g.trainer.get_params(0) if g.rank == world - 1 else None
    g.close()
    return losses, final
