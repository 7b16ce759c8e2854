"""Summarise an `ncu --metrics gpu__time_duration.sum --csv` launch list: per-kernel shares."""
import collections
import csv
import re
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
    return data


def short(name):
    name = re.sub(r"\(.*", "", name)
    for p in ("void ", "tmgx::", "(anonymous namespace)::", "unnamed>::"):
        name = name.replace(p, "")
    return name


def main(path, top=25):
    data = load(path)
    scale = {"nsecond": 1e-3, "usecond": 1.0, "msecond": 1e3, "ns": 1e-3, "us": 1.0, "ms": 1e3}
    tot = collections.defaultdict(float)
    cnt = collections.Counter()
    for d in data:
        k = short(d["Kernel Name"]) + " " + d["Grid Size"]
        tot[k] += float(d["Metric Value"]) * scale.get(d["Metric Unit"], 1e-3)
        cnt[k] += 1
    s = sum(tot.values())
    print(f"{len(data)} launches, total {s/1e3:.3f} ms (cold-cache, serialised)")
    for k, v in sorted(tot.items(), key=lambda x: -x[1])[:top]:
        print(f"{100*v/s:5.1f}%  {v/1e3:8.3f} ms  x{cnt[k]:<4d} {k}")


if __name__ == "__main__":
    main(sys.argv[1], int(sys.argv[2]) if len(sys.argv) > 2 else 25)
