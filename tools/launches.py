"""Summarise an ncu --metrics gpu__time_duration.sum --csv launch list (per-kernel totals)."""
import collections
import csv
import sys

def main(path, passes=6, drop_prefix=("void at::", "at::")):
    rows = list(csv.reader(open(path)))
    hi = [i for i, r in enumerate(rows) if 'Kernel Name' in r][0]
    h = rows[hi]
    ki, vi, ui = h.index('Kernel Name'), h.index('Metric Value'), h.index('Metric Unit')
    agg = collections.defaultdict(lambda: [0, 0.0])
    for r in rows[hi + 1:]:
        if len(r) <= vi:
            continue
        v = float(r[vi].replace(',', ''))
        v = v / 1e3 if r[ui] == 'ns' else (v * 1e3 if r[ui] == 'ms' else v)
        name = r[ki].split('(')[0][:70]
        if name.startswith(drop_prefix):
            continue
        agg[name][0] += 1
        agg[name][1] += v
    tot = sum(v[1] for v in agg.values())
    print(f"# {path}: per-pass ms assumes {passes} identical passes; cold-cache serialised launches")
    print("# ms/pass  share  launches/pass  avg_us  kernel")
    for k, (n, t) in sorted(agg.items(), key=lambda x: -x[1][1]):
        print(f"{t / 1e3 / passes:8.3f} {100 * t / tot:5.1f}% {n / passes:7.1f} {t / n:10.1f}  {k}")
    print(f"# total {tot / 1e3 / passes:.3f} ms/pass")

if __name__ == "__main__":
    main(sys.argv[1], int(sys.argv[2]) if len(sys.argv) > 2 else 6)
