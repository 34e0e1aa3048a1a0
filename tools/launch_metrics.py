"""Per-kernel summary of an ncu --csv launch list with several metrics
(gpu__time_duration.sum plus optional dram__bytes_read/write.sum)."""
import collections
import csv
import sys


def main(path):
    rows = list(csv.reader(open(path)))
    hdr, data = None, []
    for r in rows:
        if r and r[0] == "ID":
            hdr = r
            continue
        if hdr and len(r) == len(hdr):
            data.append(dict(zip(hdr, r)))
    agg = collections.defaultdict(lambda: collections.defaultdict(list))
    for d in data:
        agg[d["Kernel Name"][:48]][d["Metric Name"]].append(float(d["Metric Value"].replace(",", "")))
    tot = sum(sum(v["gpu__time_duration.sum"]) for v in agg.values())
    for k, v in sorted(agg.items(), key=lambda kv: -sum(kv[1]["gpu__time_duration.sum"])):
        t = v["gpu__time_duration.sum"]
        n = len(t)
        avg = sum(t) / n
        rd = sum(v.get("dram__bytes_read.sum", [0])) / n
        wr = sum(v.get("dram__bytes_write.sum", [0])) / n
        print(f"{k:50s} n={n:5d} avg={avg / 1000:9.2f} us share={sum(t) / tot * 100:5.1f}% "
              f"dram={(rd + wr) / 1e6:8.1f} MB  {(rd + wr) / avg:6.0f} GB/s")


if __name__ == "__main__":
    main(sys.argv[1])
