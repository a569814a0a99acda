"""Quick timing probe of the ResNet CDP step on one GPU (development tool, not the bench).
env: CDP_ARCH=resnet18|resnet50 (not ARCH: the ncu launcher script overwrites it)  MB  DT  STEPS  PROFILE=1 (per-kernel table from the instrumented step)"""
import collections, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
from paper_2403_08837_b200.resnet import DeviceResNet, synthetic_cifar, RESNET18, RESNET50, layer_specs

arch = os.environ.get("CDP_ARCH", "resnet18")
cfg = dict(RESNET18) if arch == "resnet18" else dict(RESNET50)
hw, classes = (32, 10) if arch == "resnet18" else (224, 1000)
B = int(os.environ.get("MB", "128"))
dtype = os.environ.get("DT", "bf16")
steps = int(os.environ.get("STEPS", "20"))
x, y = synthetic_cifar(2 * B, hw=hw, classes=classes)
tr = DeviceResNet(cfg["widths"], cfg["depths"], micro_batch=B, dtype=dtype, momentum=0.9, inputs=x, labels=y,
                  image_hw=hw, classes=classes, block=cfg["block"], stem=cfg["stem"])
specs = layer_specs(cfg["widths"], cfg["depths"], 3, hw, cfg["block"], cfg["stem"], classes)
rng = np.random.default_rng(0)
theta = np.concatenate([rng.normal(0, (2.0 / (np.prod(s[:3]) if k == "conv" else s[0])) ** 0.5, size=int(np.prod(s)))
                        if k != "bn" else np.concatenate([np.ones(s[0] // 2), np.zeros(s[0] // 2)])
                        for k, s, _ in specs])
tr.set_params(theta, -1)
tr.connect([tr.region()])
GEMM_NAMES = {"conv_fprop", "conv_fprop_1x1", "conv_dgrad", "conv_dgrad_1x1", "conv_dgrad_s2", "conv_wgrad_hop",
              "conv_wgrad_hop_1x1", "stem_fprop", "stem_wgrad_hop"}
if os.environ.get("ONLY"):  # one eager instrumented step only (for ncu --launch-skip over gemm_pk launches)
    ops = tr.profile_step(rng.permutation(len(x))[:B], 0.05, serial=True)
    gi = 0
    for i, (name, fl, by, t) in enumerate(ops):
        if name in GEMM_NAMES:
            print(f"gemm_pk {gi} op {i} {name} {t * 1e3:.1f} us")
            gi += 1
    sys.exit(0)
for k in range(3):
    tr.step(rng.permutation(len(x))[:B], 0.05)
tr.sync()
ms = []
for k in range(steps):
    tr.flush_l2(); tr.mark(0); tr.step(rng.permutation(len(x))[:B], 0.05); tr.mark(1)
    ms.append(tr.elapsed(0, 1))
st = tr.stats()
med = float(np.median(ms))
print(f"{arch} B={B} {dtype}: step ms median {med:.3f} samples/s {B / med * 1e3:.0f}  "
      f"tensor TFLOP/s {st['tensor_flops_per_step'] / med / 1e9:.1f}  {st}")
print("losses", tr.history(steps + 3)[0][-5:])
if os.environ.get("PROFILE"):
    agg = collections.defaultdict(lambda: [0, 0.0, 0.0, 0.0])
    ops = tr.profile_step(rng.permutation(len(x))[:B], 0.05, serial=True)
    for name, fl, by, t in ops:
        a = agg[name]; a[0] += 1; a[1] += t; a[2] += fl; a[3] += by
    tot = sum(a[1] for a in agg.values())
    print(f"instrumented step: sum of kernel times {tot:.3f} ms over {len(ops)} launches")
    for name, a in sorted(agg.items(), key=lambda kv: -kv[1][1]):
        rate = f"{a[2] / a[1] / 1e9:8.1f} TFLOP/s" if a[2] else f"{a[3] / a[1] / 1e6:8.1f} GB/s"
        print(f"  {name:24s} n={a[0]:4d} {a[1]:8.3f} ms {100 * a[1] / tot:5.1f}%  {rate}")
    if os.environ.get("TOP"):
        print("top launches:")
        for i, (name, fl, by, t) in sorted(enumerate(ops), key=lambda kv: -kv[1][3])[:int(os.environ["TOP"])]:
            rate = f"{fl / t / 1e9:8.1f} TFLOP/s" if fl else f"{by / t / 1e6:8.1f} GB/s"
            print(f"  #{i:4d} {name:24s} {t * 1e3:8.1f} us  {rate}  flops {fl:.3g} bytes {by:.3g}")
    if os.environ.get("OPS"):  # every launch of the named classes (comma-separated), in step order
        want = set(os.environ["OPS"].split(","))
        for i, (name, fl, by, t) in enumerate(ops):
            if name in want:
                print(f"  #{i:4d} {name:24s} {t * 1e3:8.1f} us  {by / 1e6:8.2f} MB  {by / t / 1e6:8.1f} GB/s")
