import numpy as np, sys
sys.path.insert(0, '.')
from oracle import engine as OE
from paper_2403_08837_b200.device import DeviceMlpTrainer
from paper_2403_08837_b200.rules import min_delay_rule, max_delay_rule
from paper_2403_08837_b200.training import make_mlp_task

task = make_mlp_task(n=4, micro_batch_size=4, seed=5, width=8, in_dim=6, out_dim=3, loss_kind="xent")
ot = OE.make_mlp_task(n=4, micro_batch_size=4, seed=5, width=8, in_dim=6, out_dim=3, loss_kind="xent")
for rname, rule in (("v1", max_delay_rule(4)), ("v2", min_delay_rule(4))):
    tr = DeviceMlpTrainer(task.model.dims, 4, 4, 1, rule, dtype="fp32", inputs=task.inputs, targets=task.targets)
    init = np.concatenate(task.init_params())
    tr.set_params(init, -1)
    cur = task.init_params(); prev = [p.copy() for p in cur]
    fresh = OE.fresh_table("cdp-v2" if rname == "v2" else "cdp-v1", 4)
    for t in range(1, 5):
        tr.step(task.permutation(t), 0.05)
        tr.sync()
        new, loss = OE.advance(ot, cur, prev, t, ot.micro_batches(t), 0.05, fresh)
        prev, cur = cur, new
        g0 = tr.get_params(0); g1 = tr.get_params(1)
        l, f = tr.history(1)
        e0 = np.abs(g0 - np.concatenate(cur)).max(); e1 = np.abs(g1 - np.concatenate(prev)).max()
        print(rname, t, "loss", l[-1], loss, "cur err", e0, "prev err", e1)
        # per stage errors
        sizes = task.model.stage_sizes
        b = np.cumsum((0,)+sizes)
        print("   stage cur errs", [float(np.abs(g0[b[k]:b[k+1]] - np.concatenate(cur)[b[k]:b[k+1]]).max()) for k in range(4)])
