"""Summarise an ncu --metrics gpu__time_duration.sum --csv launch list (our kernels only)."""
import collections
import csv
import io
import re
import sys


def load(path):
    txt = open(path).read().split("\n")
    start = next(i for i, l in enumerate(txt) if l.startswith('"ID"'))
    return list(csv.DictReader(io.StringIO("\n".join(txt[start:]))))


def summarise(path, per_step=None, prefix="cabsk"):
    rows = [r for r in load(path) if prefix in r["Kernel Name"]]
    if per_step:
        rows = rows[-per_step:]
    agg = collections.OrderedDict()
    tot = 0.0
    for r in rows:
        nm = re.sub(r"\(.*", "", r["Kernel Name"]).replace("void cabsk::", "")
        t = float(r["Metric Value"])
        a = agg.setdefault(nm, [0, 0.0])
        a[0] += 1
        a[1] += t
        tot += t
    out = []
    for k, (c, t) in sorted(agg.items(), key=lambda x: -x[1][1]):
        out.append(f"{k:48s} {c:5d} launches {t / 1e3:10.1f} us  {100 * t / tot:5.1f}%")
    out.append(f"total {len(rows)} launches {tot / 1e3:.1f} us")
    return "\n".join(out)


if __name__ == "__main__":
    print(summarise(sys.argv[1], int(sys.argv[2]) if len(sys.argv) > 2 else None))
