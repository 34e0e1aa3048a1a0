"""Summarise an ncu --csv launch list (gpu__time_duration.sum) by kernel."""
import collections
import csv
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


def main(path):
    data = load(path)
    agg = collections.defaultdict(list)
    for d in data:
        name = d["Kernel Name"].split("(")[0][:70]
        agg[name].append(float(d["Metric Value"]))
    tot = sum(sum(v) for v in agg.values())
    print(f"{len(data)} launches, {tot / 1000:.1f} us total")
    for k, v in sorted(agg.items(), key=lambda x: -sum(x[1])):
        print(f"{k:70s} n={len(v):4d} avg={sum(v) / len(v) / 1000:9.2f} us share={sum(v) / tot:6.1%}")


if __name__ == "__main__":
    main(sys.argv[1])
