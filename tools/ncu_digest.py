"""Digest of an ncu capture exported as CSV (details / raw / sass pages) — development tool.
usage: python tools/ncu_digest.py <prefix> [top]   (reads <prefix>_details.csv, _raw.csv, _sass.csv.gz)"""
import csv, gzip, sys

pre = sys.argv[1]
top = int(sys.argv[2]) if len(sys.argv) > 2 else 14
rows = list(csv.reader(open(pre + "_details.csv")))
h = rows[0]
im, iv, iu = h.index("Metric Name"), h.index("Metric Value"), h.index("Metric Unit")
print(rows[1][h.index("Kernel Name")][:100], rows[1][h.index("Grid Size")], rows[1][h.index("Block Size")])
want = ["Duration", "DRAM Throughput", "Memory Throughput", "L2 Cache Throughput", "Compute (SM) Throughput",
        "Issue Slots Busy", "Registers Per Thread", "Achieved Occupancy", "Eligible Warps Per Scheduler",
        "Warp Cycles Per Issued Instruction"]
seen = set()
for r in rows[1:]:
    if r[im] in want and r[im] not in seen:
        seen.add(r[im])
        print(f"  {r[im]:40s} {r[iv]:>12s} {r[iu]}")
raw = list(csv.reader(open(pre + "_raw.csv")))
d = dict(zip(raw[0], raw[2]))
for k in ("dram__bytes_read.sum", "dram__bytes_write.sum"):
    print(f"  {k:40s} {d.get(k, '?'):>12s} {raw[1][raw[0].index(k)] if k in raw[0] else ''}")
lines = gzip.open(pre + "_sass.csv.gz", "rt").read().splitlines()
srows = list(csv.reader(lines[1:]))
sh = srows[0]
sc = [i for i, x in enumerate(sh) if x.startswith("stall_") and "Not Issued" not in x]
tot = sum(float(r[2] or 0) for r in srows[1:]) or 1.0
agg = {}
for r in srows[1:]:
    for i in sc:
        agg[sh[i]] = agg.get(sh[i], 0) + float(r[i] or 0)
print("  stalls:", ", ".join(f"{k[6:]} {v / tot * 100:.1f}%" for k, v in sorted(agg.items(), key=lambda kv: -kv[1])[:8]))
for r in sorted(srows[1:], key=lambda r: -float(r[2] or 0))[:top]:
    rs = max(((float(r[i] or 0), sh[i][6:]) for i in sc))
    print(f"  {float(r[2]) / tot * 100:5.1f}% {r[1].strip()[:64]:64s} {rs[1]}")
