"""Summarise an ncu --metrics gpu__time_duration.sum launch list: per kernel, launches,
total and share of the (serialised, cold-cache) kernel time."""
import collections
import csv
import sys


def main(path, out):
    rows = list(csv.reader(open(path)))
    hdr = None
    tot = collections.OrderedDict()
    for r in rows:
        if "Kernel Name" in r:
            hdr = r
            continue
        if not hdr or len(r) != len(hdr):
            continue
        d = dict(zip(hdr, r))
        if d.get("Metric Name") != "gpu__time_duration.sum":
            continue
        name = d["Kernel Name"].split("(")[0].replace("void ", "")
        v = float(d["Metric Value"].replace(",", ""))
        unit = d.get("Metric Unit", "ns")
        v *= {"ns": 1e-3, "nsecond": 1e-3, "us": 1.0, "usecond": 1.0, "ms": 1e3, "msecond": 1e3}.get(unit, 1e-3)
        c = tot.setdefault(name, [0, 0.0])
        c[0] += 1
        c[1] += v
    allt = sum(v[1] for v in tot.values())
    lines = [f"{'kernel':60s} {'launches':>8s} {'total_us':>10s} {'share':>6s}"]
    for k, (n, t) in sorted(tot.items(), key=lambda kv: -kv[1][1]):
        lines.append(f"{k[:60]:60s} {n:8d} {t:10.1f} {100 * t / allt:5.1f}%")
    lines.append(f"{'TOTAL':60s} {sum(v[0] for v in tot.values()):8d} {allt:10.1f}")
    open(out, "w").write("\n".join(lines) + "\n")
    print("\n".join(lines))


if __name__ == "__main__":
    main(sys.argv[1], sys.argv[2])
