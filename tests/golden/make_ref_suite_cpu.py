"""Generate tests/golden/ref_suite_cpu.json: the pass / fail outcome of the
reference's own test suite (/root/reference/proj/tests: unit tests and the
acceptance criteria C01-C10) built against the REFERENCE's headers on the CPU
(`make -C tests/refsuite cpu`).  tests/test_gpu_refsuite.py runs the same test
files built against this repository's drop-in headers on the B200 and compares
with this baseline.  Run here (the reference exists only in this container):

    python tests/golden/make_ref_suite_cpu.py
"""
import json
import os
import re
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, os.path.join(ROOT, "tests"))
from refsuite_parse import parse  # noqa: E402


def main():
    subprocess.run(["make", "-s", "-C", os.path.join(ROOT, "tests", "refsuite"), "cpu"], check=True)
    exe = os.path.join(ROOT, "tests", "refsuite", "_build", "ref_suite_cpu")
    r = subprocess.run([exe], capture_output=True, text=True, cwd="/tmp", timeout=1800)
    out = parse(r.stdout)
    out["generator"] = "tests/golden/make_ref_suite_cpu.py (reference headers, g++ -O3, CPU)"
    out["threads"] = os.cpu_count()
    with open(os.path.join(HERE, "ref_suite_cpu.json"), "w") as f:
        json.dump(out, f, indent=1, sort_keys=True)
    print(f"{len(out['passed'])} passed, {len(out['failed'])} failed: {out['failed']}")


if __name__ == "__main__":
    main()
