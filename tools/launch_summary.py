"""Summarise an ncu launch list (gpu__time_duration.sum [+ launch__grid_size]) per kernel:
launches, mean duration, share of captured time, and SM-time (duration x CTAs
resident, capped at 148) -- the throughput cost when lanes overlap kernels."""
import collections
import csv
import io
import re
import sys


def main(path):
    txt = open(path).read()
    txt = txt[txt.index('"ID"'):]
    agg = collections.OrderedDict()
    for r in csv.DictReader(io.StringIO(txt)):
        if r["Metric Name"] != "gpu__time_duration.sum":
            continue
        name = r["Kernel Name"]
        m = re.search(r"(\w+_kernel)(<[^(]*>)?", name)
        key = ((m.group(1) + (m.group(2) or "")[:40]) if m else name[:40], r["Grid Size"], r["Block Size"])
        a = agg.setdefault(key, [0, 0.0])
        a[0] += 1
        a[1] += float(r["Metric Value"].replace(",", ""))
    tot = sum(v[1] for v in agg.values())
    print("| kernel | grid | block | launches | mean us | share | SM-us/launch |")
    print("|---|---|---|---|---|---|---|")
    for (k, g, b), (n, t) in sorted(agg.items(), key=lambda kv: -kv[1][1]):
        dims = [int(x) for x in re.findall(r"\d+", g)]
        ctas = 1
        for d in dims:
            ctas *= d
        us = t / n / 1000
        print(f"| `{k}` | {g} | {b} | {n} | {us:.1f} | {t / tot:.3f} | {us * min(ctas, 148):.0f} |")


if __name__ == "__main__":
    main(sys.argv[1])
