"""Summarise an `ncu --metrics gpu__time_duration.sum --csv` launch list as
markdown: per kernel, launches, total and mean ms, and the share of the hot
path's time (the kernels a bench step launches).  usage: launch_summary.py CSV"""
import collections
import csv
import sys

UNIT = {"nsecond": 1e-6, "ns": 1e-6, "usecond": 1e-3, "us": 1e-3, "msecond": 1.0, "ms": 1.0, "second": 1e3}


def main(path):
    rows = list(csv.reader(open(path)))
    hdr, data = None, []
    for r in rows:
        if r and r[0] == "ID":
            hdr = r
            continue
        if hdr and len(r) == len(hdr):
            data.append(dict(zip(hdr, r)))
    agg = collections.OrderedDict()
    for d in data:
        name = d["Kernel Name"]
        short = name.split("(")[0].replace("void ", "").replace("atos::", "")
        ms = float(d["Metric Value"].replace(",", "")) * UNIT.get(d["Metric Unit"], 1e-6)
        agg.setdefault(short, []).append(ms)
    tot = sum(sum(v) for v in agg.values())
    print(f"{len(data)} launches, {tot:.1f} ms of kernel time in the whole command\n")
    print("| kernel | launches | total ms | mean ms / launch | share of all kernel time |")
    print("|---|---|---|---|---|")
    for k, v in sorted(agg.items(), key=lambda x: -sum(x[1])):
        print(f"| `{k[:110]}` | {len(v)} | {sum(v):.3f} | {sum(v) / len(v):.4f} | {100 * sum(v) / tot:.2f}% |")


if __name__ == "__main__":
    main(sys.argv[1])
