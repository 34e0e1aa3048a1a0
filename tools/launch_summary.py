"""Summarise an ncu --csv launch list by kernel: time (gpu__time_duration.sum),
and, when captured, DRAM bytes (dram__bytes_read.sum + dram__bytes_write.sum)."""
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
    launches = collections.OrderedDict()  # ID -> {name, metrics}
    for d in data:
        e = launches.setdefault(d["ID"], {"name": d["Kernel Name"].split("(")[0][:70], "m": {}})
        e["m"][d["Metric Name"]] = float(d["Metric Value"].replace(",", ""))
    agg = collections.defaultdict(lambda: [0, 0.0, 0.0])
    for e in launches.values():
        a = agg[e["name"]]
        a[0] += 1
        a[1] += e["m"].get("gpu__time_duration.sum", 0.0)
        a[2] += e["m"].get("dram__bytes_read.sum", 0.0) + e["m"].get("dram__bytes_write.sum", 0.0)
    tot = sum(v[1] for v in agg.values()) or 1.0
    print(f"{len(launches)} launches, {tot / 1000:.1f} us total")
    for k, (n, t, b) in sorted(agg.items(), key=lambda x: -x[1][1]):
        extra = f" dram/launch={b / n / 1e6:8.1f} MB {b / (t * 1e-9) / 1e9:6.0f} GB/s" if b else ""
        print(f"{k:70s} n={n:5d} avg={t / n / 1000:9.2f} us share={t / tot:6.1%}{extra}")


if __name__ == "__main__":
    main(sys.argv[1])
