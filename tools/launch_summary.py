"""Summarise an `ncu --metrics gpu__time_duration.sum --csv` launch list:
per-kernel launches, total time and share of all device time."""

import collections
import csv
import json
import sys


def summarise(path):
    rows = list(csv.reader(open(path)))
    hi = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
    h = rows[hi]
    ki, vi, ui = h.index("Kernel Name"), h.index("Metric Value"), h.index("Metric Unit")
    scale = {"ns": 1e-6, "nsecond": 1e-6, "us": 1e-3, "usecond": 1e-3, "ms": 1.0, "msecond": 1.0}
    tot = collections.defaultdict(lambda: [0, 0.0])
    for r in rows[hi + 1:]:
        if len(r) <= vi:
            continue
        name = r[ki].replace("(anonymous namespace)::", "").replace("<unnamed>::", "")
        name = name.replace("void ", "").replace("vpg::", "").replace("CUB_200802_SM_1000::", "cub::")
        name = name.split("(")[0]
        if name.startswith("cub::") or name.startswith("at::"):
            name = name.split("<")[0]
        tot[name][0] += 1
        tot[name][1] += float(r[vi].replace(",", "")) * scale[r[ui]]
    total = sum(v for _, v in tot.values())
    out = [{"kernel": k, "launches": c, "total_ms": round(v, 4), "share": round(v / total, 4)}
           for k, (c, v) in sorted(tot.items(), key=lambda kv: -kv[1][1])]
    return {"total_ms": total, "kernels": out}


if __name__ == "__main__":
    s = summarise(sys.argv[1])
    if len(sys.argv) > 2:
        json.dump(s, open(sys.argv[2], "w"), indent=1)
    for k in s["kernels"][:30]:
        print(f"{k['kernel']:48s} {k['launches']:6d} {k['total_ms']:10.3f} ms {100*k['share']:5.1f}%")
    print("total ms", round(s["total_ms"], 3))
