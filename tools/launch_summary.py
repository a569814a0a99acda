"""Summarise an `ncu --metrics gpu__time_duration.sum --csv` launch list (last `--last` launches)."""
import collections, csv, io, re, sys

def load(path):
    txt = open(path).read().splitlines()
    start = next(i for i, l in enumerate(txt) if l.startswith('"ID"'))
    rows = list(csv.DictReader(io.StringIO("\n".join(txt[start:]))))
    out = []
    for r in rows:
        if r['Metric Name'] != 'gpu__time_duration.sum':
            continue
        v = float(r['Metric Value'].replace(',', ''))
        u = r['Metric Unit']
        us = v / 1000 if u in ('ns', 'nsecond') else v if u in ('us', 'usecond') else v * 1000
        out.append((r['Kernel Name'], r['Grid Size'], us))
    return out

if __name__ == "__main__":
    path = sys.argv[1]
    last = int(sys.argv[2]) if len(sys.argv) > 2 else 0
    grid = "--grid" in sys.argv
    rows = load(path)
    if last:
        rows = rows[-last:]
    agg = collections.defaultdict(lambda: [0, 0.0])
    for name, g, us in rows:
        k = re.sub(r'\(.*', '', name.replace('(anonymous namespace)::', ''))[:100] + (f" grid{g}" if grid else "")
        agg[k][0] += 1
        agg[k][1] += us
    tot = sum(v[1] for v in agg.values())
    print(f"| kernel | launches | total us | share |\n|---|---|---|---|")
    for k, v in sorted(agg.items(), key=lambda kv: -kv[1][1])[:40]:
        print(f"| `{k}` | {v[0]} | {v[1]:.1f} | {100 * v[1] / tot:.1f}% |")
    print(f"\ntotal {tot:.1f} us over {len(rows)} launches")
