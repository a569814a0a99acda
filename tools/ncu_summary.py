"""Key numbers of one-kernel `ncu --set full` reports (duration, DRAM bytes, tensor-pipe and SM utilisation)."""
import csv, io, json, subprocess, sys

KEYS = {
    "gpu__time_duration.sum": "duration",
    "dram__bytes_read.sum": "dram_read",
    "dram__bytes_write.sum": "dram_write",
    "sm__ops_path_tensor_op_utchmma_src_bf16_dst_fp32_sparsity_off.sum.pct_of_peak_sustained_elapsed": "tensor_pct",
    "sm__throughput.avg.pct_of_peak_sustained_elapsed": "sm_pct",
    "dram__throughput.avg.pct_of_peak_sustained_elapsed": "dram_pct",
    "lts__t_bytes.sum": "l2_bytes",
    "launch__grid_size": "grid",
    "launch__registers_per_thread": "regs",
}
SCALE = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "us": 1e-6, "ns": 1e-9, "ms": 1e-3, "s": 1, "%": 1, "": 1}


def summary(path):
    out = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    h, u, v = rows[0], rows[1], rows[2]
    d = {"kernel": v[h.index("Kernel Name")]}
    for name, unit, val in zip(h, u, v):
        if name in KEYS:
            try:
                d[KEYS[name]] = float(val.replace(",", "")) * SCALE.get(unit, 1)
            except ValueError:
                pass
    return d


if __name__ == "__main__":
    for p in sys.argv[1:]:
        print(json.dumps({p: summary(p)}))
