"""DRAM traffic per kernel class of one serialised training step (development tool, run under ncu).

  ncu --profile-from-start off --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum \
      --csv --log-file gpurun_out/<m>_traffic.csv python tools/step_traffic.py <model> gpurun_out/<m>_ops.json
  python tools/step_traffic.py --join gpurun_out/<m>_ops.json gpurun_out/<m>_traffic.csv

The step runs between cudaProfilerStart/Stop, so ncu's launch list is exactly the step's op list
(one kernel per op, in order); --join sums DRAM bytes per op name and writes the per-launch average of
each class (the `traffic` figure of bench.py's roofline) to stdout as JSON.
"""
import csv, io, json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def run(model, out):
    import numpy as np
    import torch
    from paper_2403_08837_b200.resnet import DeviceResNet, synthetic_cifar, RESNET18, RESNET50, layer_specs
    rng = np.random.default_rng(0)
    if model == "vit_b16":
        from paper_2403_08837_b200.vit import VIT_B16, DeviceVit
        from oracle.vit_torch import init_flat
        B = 32
        x, y = synthetic_cifar(2 * B, hw=224, classes=1000)
        tr = DeviceVit(dict(VIT_B16), B, momentum=0.9, inputs=x, labels=y)
        tr.set_params(init_flat(**VIT_B16, seed=0), -1)
        lr = 0.01
    else:
        cfg = dict(RESNET18) if model == "resnet18" else dict(RESNET50)
        hw, classes = (32, 10) if model == "resnet18" else (224, 1000)
        B = 128
        x, y = synthetic_cifar(2 * B, hw=hw, classes=classes)
        tr = DeviceResNet(cfg["widths"], cfg["depths"], micro_batch=B, dtype="bf16", momentum=0.9, inputs=x,
                          labels=y, image_hw=hw, classes=classes, block=cfg["block"], stem=cfg["stem"])
        specs = layer_specs(cfg["widths"], cfg["depths"], 3, hw, cfg["block"], cfg["stem"], classes)
        theta = np.concatenate([rng.normal(0, (2.0 / (np.prod(s[:3]) if k == "conv" else s[0])) ** 0.5,
                                           size=int(np.prod(s))) if k != "bn" else
                                np.concatenate([np.ones(s[0] // 2), np.zeros(s[0] // 2)]) for k, s, _ in specs])
        tr.set_params(theta, -1)
        lr = 0.05
    tr.connect([tr.region()])
    tr.step(rng.permutation(len(x))[:B], lr)
    tr.sync()
    torch.cuda.synchronize()
    torch.cuda.profiler.start()
    ops = tr.profile_step(rng.permutation(len(x))[:B], lr, serial=True)
    torch.cuda.synchronize()
    torch.cuda.profiler.stop()
    with open(out, "w") as fh:
        json.dump([[n, fl, by] for n, fl, by, _t in ops], fh)


def join(ops_path, csv_path):
    ops = json.load(open(ops_path))
    text = open(csv_path).read()
    rows = list(csv.DictReader(io.StringIO(text[text.index('"ID"'):])))
    per = {}
    for r in rows:
        k = int(r["ID"])
        v = float(r["Metric Value"].replace(",", ""))
        unit = r.get("Metric Unit", "")
        scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "ns": 1e-9, "us": 1e-6, "ms": 1e-3,
                 "s": 1.0}[unit]
        d = per.setdefault(k, {"kernel": r["Kernel Name"]})
        d[r["Metric Name"]] = v * scale
    launches = [per[k] for k in sorted(per)]
    if len(launches) != len(ops):
        raise SystemExit(f"launch count {len(launches)} != op count {len(ops)}")
    agg = {}
    for (name, fl, by), l in zip(ops, launches):
        name = name.split("\0", 1)[0].strip()
        a = agg.setdefault(name, {"launches": 0, "dram_bytes": 0.0, "duration_s": 0.0, "algorithmic_flops": 0.0,
                                  "algorithmic_bytes": 0.0, "kernels": set()})
        a["launches"] += 1
        a["dram_bytes"] += l.get("dram__bytes_read.sum", 0.0) + l.get("dram__bytes_write.sum", 0.0)
        a["duration_s"] += l.get("gpu__time_duration.sum", 0.0)
        a["algorithmic_flops"] += fl
        a["algorithmic_bytes"] += by
        a["kernels"].add(l["kernel"].split("(")[0])
    out = {}
    for name, a in agg.items():
        n = a["launches"]
        out[name] = {"launches": n, "dram_bytes_per_launch": a["dram_bytes"] / n,
                     "algorithmic_flops_per_launch": a["algorithmic_flops"] / n,
                     "algorithmic_bytes_per_launch": a["algorithmic_bytes"] / n,
                     "ncu_us_per_launch": a["duration_s"] / n * 1e6, "kernels": sorted(a["kernels"])}
    return out


if __name__ == "__main__":
    if sys.argv[1] == "--join":
        print(json.dumps(join(sys.argv[2], sys.argv[3]), indent=1))
    else:
        run(sys.argv[1], sys.argv[2])
