"""Parse the output of a GoogleTest-style run (tests/refsuite shim)."""
import re


def parse(text: str) -> dict:
    passed, failed = [], []
    for m in re.finditer(r"^\[ +(OK|FAILED) +\] (\S+\.\S+)$", text, flags=re.M):
        (passed if m.group(1) == "OK" else failed).append(m.group(2))
    acc = {}
    for m in re.finditer(r"^\[ACCEPTANCE\] #(\d+) ([^:]+): (PASS|FAIL|WARN) \((.*)\)$", text, flags=re.M):
        acc[f"C{int(m.group(1)):02d}"] = {"name": m.group(2), "status": m.group(3), "detail": m.group(4)}
    c01 = acc.get("C01", {}).get("detail", "")
    m = re.search(r"ranks (\d+)/(\d+), errors@1e-10 (\d+)/(\d+)", c01)
    if m:
        acc["C01"]["ranks_ok"], acc["C01"]["cells"], acc["C01"]["errors_ok"] = int(m.group(1)), int(m.group(2)), int(m.group(3))
        acc["C01"]["failing_cells"] = re.findall(r"\[(\S+ t\d+ rmax=-?\d+ eps=[0-9.e-]+)", c01)
    return {"passed": sorted(set(passed)), "failed": sorted(set(failed)), "acceptance": acc}
