"""Summarise an ncu launch list (--metrics gpu__time_duration.sum --csv) into
per-kernel counts, mean duration and share of the captured time."""

import collections
import csv
import io
import re
import sys


def summarize(path: str) -> str:
    txt = open(path).read()
    txt = txt[txt.index('"ID"'):]
    agg = collections.OrderedDict()
    for r in csv.DictReader(io.StringIO(txt)):
        name = r["Kernel Name"]
        m = re.search(r"(gemm_simt_kernel<amun::(\w+)>|splitk_reduce_kernel<amun::(\w+)>|logits_tc_kernel|\w+_kernel)", name)
        key = (m.group(0) if m else name[:48], r["Grid Size"])
        a = agg.setdefault(key, [0, 0.0])
        a[0] += 1
        a[1] += float(r["Metric Value"])
    tot = sum(v[1] for v in agg.values())
    out = ["| kernel | grid | launches | mean us | share |", "|---|---|---|---|---|"]
    for (k, g), (n, t) in sorted(agg.items(), key=lambda kv: -kv[1][1]):
        out.append(f"| `{k}` | {g} | {n} | {t / n / 1000:.1f} | {t / tot:.3f} |")
    return "\n".join(out)


if __name__ == "__main__":
    print(summarize(sys.argv[1]))
