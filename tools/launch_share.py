"""Per-kernel totals and shares from an ncu --metrics gpu__time_duration.sum CSV launch list."""
import collections
import csv
import sys

UNITS = {"ns": 1e-3, "nsecond": 1e-3, "us": 1.0, "usecond": 1.0, "ms": 1e3, "msecond": 1e3}


def shares(path):
    rows = [r for r in csv.reader(open(path)) if len(r) > 10]
    hdr = rows[0]
    ci = {h: i for i, h in enumerate(hdr)}
    tot, cnt = collections.Counter(), collections.Counter()
    for r in rows[1:]:
        if r[ci["Metric Name"]] != "gpu__time_duration.sum":
            continue
        k = r[ci["Kernel Name"]].split("(")[0]
        v = float(r[ci["Metric Value"]].replace(",", "")) * UNITS[r[ci["Metric Unit"]]]
        tot[k] += v
        cnt[k] += 1
    return tot, cnt


if __name__ == "__main__":
    tot, cnt = shares(sys.argv[1])
    T = sum(tot.values())
    print(f"{'kernel':70s} {'launches':>8s} {'total us':>10s} {'mean us':>9s} {'share':>6s}")
    for k, v in tot.most_common():
        print(f"{k[:70]:70s} {cnt[k]:8d} {v:10.1f} {v / cnt[k]:9.1f} {v / T * 100:5.1f}%")
