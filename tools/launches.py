"""Summarise an ncu --metrics gpu__time_duration.sum CSV launch list per kernel."""
import collections
import csv
import sys


def summarize(path, encodes=1):
    rows = list(csv.reader(open(path)))
    hdr, data = None, []
    for r in rows:
        if r and r[0] == "ID":
            hdr = r
            continue
        if hdr and len(r) == len(hdr):
            data.append(dict(zip(hdr, r)))
    agg = collections.defaultdict(lambda: [0, 0.0])
    for d in data:
        if d.get("Metric Name") != "gpu__time_duration.sum":
            continue
        k = d["Kernel Name"][:60]
        agg[k][0] += 1
        agg[k][1] += float(d["Metric Value"])
    tot = sum(v[1] for v in agg.values())
    out = []
    for k, (c, t) in sorted(agg.items(), key=lambda x: -x[1][1]):
        out.append(f"{c:5d} launches {t / 1e3 / encodes:10.1f} us/encode {t / c / 1e3:9.1f} us/launch "
                   f"{100 * t / tot:5.1f}%  {k}")
    return "\n".join(out)


if __name__ == "__main__":
    print(summarize(sys.argv[1], int(sys.argv[2]) if len(sys.argv) > 2 else 1))
