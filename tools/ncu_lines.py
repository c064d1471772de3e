"""Attribute ncu warp-stall samples of one kernel to CUDA source lines.
usage: python tools/ncu_lines.py report.ncu-rep kernel_regex lib.so [topN] [ncu_kernel_regex]
(kernel_regex matches the mangled SASS section; ncu_kernel_regex, default the
same, the report's demangled kernel name)"""
import csv
import re
import subprocess
import sys
import tempfile
import os


def main():
    rep, kre, so = sys.argv[1], sys.argv[2], sys.argv[3]
    top = int(sys.argv[4]) if len(sys.argv) > 4 else 25
    nkre = sys.argv[5] if len(sys.argv) > 5 else kre
    tmp = tempfile.mkdtemp()
    subprocess.run(["cuobjdump", "-xelf", "all", os.path.abspath(so)], cwd=tmp, check=True, capture_output=True)
    cub = [f for f in os.listdir(tmp) if f.endswith(".cubin")][0]
    sass = subprocess.run(["nvdisasm", "-g", os.path.join(tmp, cub)], capture_output=True, text=True).stdout
    lines, infn, cur = {}, False, None
    for l in sass.splitlines():
        if re.search(r"\.text\.\S*" + kre, l) and "section" in l:
            infn = True
            continue
        if infn and re.search(r"^\s*\.section", l):
            break
        if not infn:
            continue
        m = re.search(r'//## File "([^"]+)", line (\d+)', l)
        if m:
            cur = (m.group(1).split("/")[-1], int(m.group(2)))
            continue
        m = re.search(r"/\*([0-9a-f]{4,})\*/", l)
        if m and cur:
            lines[int(m.group(1), 16)] = cur
    out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "-k", "regex:" + nkre], capture_output=True,
                         text=True).stdout
    r = list(csv.reader(out.splitlines()))
    h = r[1]
    rows = [dict(zip(h, x)) for x in r[2:] if len(x) == len(h)]
    base = int(rows[0]["Address"], 16)
    key = "Warp Stall Sampling (All Samples)"
    agg, tot = {}, 0.0
    for x in rows:
        v = float(x[key] or 0)
        tot += v
        k = lines.get(int(x["Address"], 16) - base, ("?", 0))
        agg[k] = agg.get(k, 0) + v
    for k, v in sorted(agg.items(), key=lambda z: -z[1])[:top]:
        print(f"{100 * v / tot:5.1f}%  {k[0]}:{k[1]}")


if __name__ == "__main__":
    main()
