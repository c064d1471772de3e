"""Summarise an ncu launch-list CSV (gpu__time_duration.sum per launch) as markdown."""
import collections
import csv
import sys


def main():
    src, title = sys.argv[1], sys.argv[2] if len(sys.argv) > 2 else "ncu launch list"
    rows = list(csv.reader(open(src)))
    hdr, data = None, []
    for r in rows:
        if r and r[0] == "ID":
            hdr = r
            continue
        if hdr and len(r) == len(hdr):
            data.append(dict(zip(hdr, r)))
    scale = {"nsecond": 1e-6, "usecond": 1e-3, "msecond": 1.0, "second": 1e3}
    agg, tot = collections.OrderedDict(), 0.0
    for d in data:
        t = float(d["Metric Value"]) * scale.get(d["Metric Unit"], 1e-6)
        name = d["Kernel Name"].split("(")[0].replace("void ", "")
        a = agg.setdefault(name, [0, 0.0])
        a[0] += 1
        a[1] += t
        tot += t
    print(f"# {title}\n")
    print("| kernel | launches | total ms | share |\n|---|---|---|---|")
    for k, (n, t) in sorted(agg.items(), key=lambda x: -x[1][1]):
        print(f"| {k} | {n} | {t:.3f} | {100 * t / tot:.1f}% |")
    print(f"\nTotal {tot:.2f} ms over {len(data)} launches (cold-cache, serialised: compare shares).\n")
    print("| # | kernel | grid | ms |\n|---|---|---|---|")
    for i, d in enumerate(data):
        t = float(d["Metric Value"]) * scale.get(d["Metric Unit"], 1e-6)
        print(f"| {i} | {d['Kernel Name'].split('(')[0].replace('void ', '')} | {d['Grid Size']} | {t:.3f} |")


if __name__ == "__main__":
    main()
