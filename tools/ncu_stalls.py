"""Stall-reason totals of one kernel in an ncu report (source page, SASS):
usage: python tools/ncu_stalls.py report.ncu-rep kernel_regex [top_instructions]"""
import csv
import subprocess
import sys


def main():
    rep, kre = sys.argv[1], sys.argv[2]
    top = int(sys.argv[3]) if len(sys.argv) > 3 else 15
    out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass", "-k", "regex:" + kre],
                         capture_output=True, text=True).stdout
    r = list(csv.reader(out.splitlines()))
    h = r[1]
    rows = [dict(zip(h, x)) for x in r[2:] if len(x) == len(h)]
    keys = [k for k in h if k.startswith("stall_") and "Not Issued" not in k]
    tot = {k: sum(float(x[k] or 0) for x in rows) for k in keys}
    s = sum(tot.values())
    print("stall reasons (% of samples):")
    for k, v in sorted(tot.items(), key=lambda z: -z[1])[:10]:
        print(f"  {k:24s} {100 * v / s:5.1f}%")
    print(f"top {top} instructions:")
    rows.sort(key=lambda x: -float(x["Warp Stall Sampling (All Samples)"] or 0))
    for x in rows[:top]:
        v = float(x["Warp Stall Sampling (All Samples)"] or 0)
        main_k = max(keys, key=lambda k: float(x[k] or 0))
        print(f"  {100 * v / s:5.1f}%  {x['Address'][-5:]}  {x['Source'].strip()[:60]:60s} {main_k}")


if __name__ == "__main__":
    main()
