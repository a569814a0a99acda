"""ViT timing / accuracy probe (development tool).  env: MB, STEPS, PROFILE=1, ACC=1 (small-config error margins)."""
import collections, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np

if os.environ.get("ACC"):
    import importlib.util as U
    here = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests", "test_gpu_vit.py")
    s = U.spec_from_file_location("tgv", here); T = U.module_from_spec(s); s.loader.exec_module(T)
    for world in (1, 2):
        from paper_2403_08837_b200.rules import rule_by_name
        rule = None if world == 1 else rule_by_name("cdp-v2", 2)
        init, x, y, perms, losses, final, stage = T._run(world, rule, 3)
        want, wl = T._oracle(init, x, y, perms, world, rule, stage)
        d = final - init; dw = want - init
        print(f"world {world}: update rel-L2 {np.linalg.norm(d - dw) / np.linalg.norm(dw):.3e}, "
              f"loss rel {np.max(np.abs(losses - wl) / np.abs(wl)):.3e}, losses {losses} vs {wl}")
    sys.exit(0)

from paper_2403_08837_b200.resnet import synthetic_cifar
from paper_2403_08837_b200.vit import VIT_B16, DeviceVit, vit_units
from oracle.vit_torch import init_flat

B = int(os.environ.get("MB", "32"))
steps = int(os.environ.get("STEPS", "10"))
cfg = dict(VIT_B16)
x, y = synthetic_cifar(2 * B, hw=224, classes=1000)
tr = DeviceVit(cfg, B, momentum=0.9, inputs=x, labels=y)
tr.set_params(init_flat(**cfg, seed=0), -1)
tr.connect([tr.region()])
rng = np.random.default_rng(0)
for k in range(3):
    tr.step(rng.permutation(len(x))[:B], 0.01)
tr.sync()
ms = []
for k in range(steps):
    tr.flush_l2(); tr.mark(0); tr.step(rng.permutation(len(x))[:B], 0.01); tr.mark(1)
    ms.append(tr.elapsed(0, 1))
st = tr.stats()
med = float(np.median(ms))
print(f"vit_b16 B={B}: step ms {med:.3f} samples/s {B / med * 1e3:.0f} tensor TFLOP/s "
      f"{st['tensor_flops_per_step'] / med / 1e9:.1f} {st}")
print("losses", tr.history(steps + 3)[0][-4:])
if os.environ.get("PROFILE"):
    agg = collections.defaultdict(lambda: [0, 0.0, 0.0, 0.0])
    ops = tr.profile_step(rng.permutation(len(x))[:B], 0.01, serial=True)
    for name, fl, by, t in ops:
        a = agg[name]; a[0] += 1; a[1] += t; a[2] += fl; a[3] += by
    tot = sum(a[1] for a in agg.values())
    print(f"instrumented step: {tot:.3f} ms over {len(ops)} launches")
    for name, a in sorted(agg.items(), key=lambda kv: -kv[1][1]):
        rate = f"{a[2] / a[1] / 1e9:8.1f} TFLOP/s" if a[2] else f"{a[3] / a[1] / 1e6:8.1f} GB/s"
        print(f"  {name:22s} n={a[0]:4d} {a[1]:8.3f} ms {100 * a[1] / tot:5.1f}%  {rate}")
