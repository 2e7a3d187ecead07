"""Per-step DRAM traffic and time share from an ncu launch list
(--metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum) of
`bench.py --steps 1 --warmup 1`: the second of the two encodes is the timed step."""
import collections
import csv
import json
import sys


def load(path):
    rows = list(csv.reader(open(path)))
    hdr, data = None, []
    for r in rows:
        if r and r[0] == "ID":
            hdr = r
            continue
        if hdr and len(r) == len(hdr):
            data.append(dict(zip(hdr, r)))
    launches = collections.OrderedDict()
    for d in data:
        launches.setdefault(d["ID"], {"name": d["Kernel Name"]})[d["Metric Name"]] = float(d["Metric Value"])
    return list(launches.values())


def main(path, out_json, patches, method="omp", selector="tree", family_json=None):
    ls = load(path)
    starts = [i for i, l in enumerate(ls) if "init_kernel" in l["name"]]
    step = ls[starts[-1]:] if starts else ls[len(ls) // 2:]   # last encode = the timed step
    t = sum(l.get("gpu__time_duration.sum", 0) for l in step)
    rd = sum(l.get("dram__bytes_read.sum", 0) for l in step)
    wr = sum(l.get("dram__bytes_write.sum", 0) for l in step)
    per = collections.defaultdict(lambda: [0, 0.0, 0.0])
    for l in step:
        k = l["name"].split("(")[0].replace("void ", "")[:48]
        per[k][0] += 1
        per[k][1] += l.get("gpu__time_duration.sum", 0)
        per[k][2] += l.get("dram__bytes_read.sum", 0) + l.get("dram__bytes_write.sum", 0)
    summary = {"patches": patches, "method": method, "selector": selector, "launches": len(step),
               "bytes_per_launch": rd + wr, "serialized_ns": t,
               "note": "dram bytes summed over every kernel of one staged step (ncu, cold caches, serialised)",
               "kernels": {k: {"launches": c, "time_share": tt / t, "dram_bytes": b} for k, (c, tt, b) in per.items()}}
    json.dump(summary, open(out_json, "w"), indent=1)
    print(json.dumps(summary, indent=1))
    if family_json:
        # ncu DRAM bytes per launch of each kernel family (bench.py's roofline.traffic)
        import os
        sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
        from paper_1412_0680_b200 import roofline as RL
        fam = collections.defaultdict(lambda: [0, 0.0])
        for l in step:
            f = RL.family_of(l["name"])
            fam[f][0] += 1
            fam[f][1] += l.get("dram__bytes_read.sum", 0) + l.get("dram__bytes_write.sum", 0)
        table = json.load(open(family_json)) if os.path.exists(family_json) else {}
        table[f"{selector}-{method}-{patches}"] = {f: b / c for f, (c, b) in fam.items()}
        json.dump(table, open(family_json, "w"), indent=1)


if __name__ == "__main__":
    a = sys.argv
    main(a[1], a[2], int(a[3]), a[4] if len(a) > 4 else "omp", a[5] if len(a) > 5 else "tree",
         a[6] if len(a) > 6 else None)
