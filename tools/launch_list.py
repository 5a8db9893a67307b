"""Condense an `ncu --metrics gpu__time_duration.sum --csv` launch list into per-kernel shares."""
import collections
import csv
import json
import sys

SCALE = {"ns": 1e-6, "nsecond": 1e-6, "us": 1e-3, "usecond": 1e-3, "ms": 1.0, "msecond": 1.0,
         "s": 1e3, "second": 1e3}


def condense(path):
    rows = [r for r in csv.reader(open(path)) if len(r) > 5]
    hdr = rows[0]
    ki, vi, ui = hdr.index("Kernel Name"), hdr.index("Metric Value"), hdr.index("Metric Unit")
    tot, cnt = collections.defaultdict(float), collections.Counter()
    for r in rows[1:]:
        name = r[ki].split("(")[0]
        tot[name] += float(r[vi].replace(",", "")) * SCALE.get(r[ui], 1.0)
        cnt[name] += 1
    s = sum(tot.values())
    return [{"kernel": k, "launches": cnt[k], "ms_total": round(v, 4), "share": round(v / s, 5)}
            for k, v in sorted(tot.items(), key=lambda x: -x[1])]


if __name__ == "__main__":
    print(json.dumps(condense(sys.argv[1]), indent=1))
