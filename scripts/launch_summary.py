"""Summarise an ncu --csv launch list (gpu__time_duration + dram bytes) by kernel."""
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
    k = collections.OrderedDict()
    for d in data:
        key = (d["ID"], d["Kernel Name"], d["Grid Size"])
        k.setdefault(key, {})[d["Metric Name"]] = float(d["Metric Value"].replace(",", ""))
    return list(k.items())


def main(path, last=None):
    items = load(path)
    if last:
        items = items[-int(last):]
    tot = sum(v.get("gpu__time_duration.sum", 0) for _, v in items)
    by = collections.defaultdict(lambda: [0, 0.0, 0.0])
    for (i, n, g), v in items:
        nm = n.split("(")[0].replace("void ", "")
        e = by[(nm, g)]
        e[0] += 1
        e[1] += v.get("gpu__time_duration.sum", 0)
        e[2] += v.get("dram__bytes_read.sum", 0) + v.get("dram__bytes_write.sum", 0)
    print(f"{path}: {len(items)} launches, {tot / 1e3:.1f} us total")
    for (nm, g), (c, t, b) in sorted(by.items(), key=lambda x: -x[1][1]):
        print(f"  {nm[:48]:48s} grid {g:15s} n={c:3d} total {t / 1e3:9.1f} us ({100 * t / tot:4.1f}%)"
              f" avg {t / c / 1e3:8.2f} us  dram {b / c / 1e6:8.2f} MB/launch")


if __name__ == "__main__":
    main(*sys.argv[1:])
