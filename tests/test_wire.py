"""Wire formats (SURVEY §8 f, rank 3): files written by the package (Python
mirror and the C++ drop-in header) are read by the reference's own
load_tt / load_tensor and vice versa, byte for byte (storage.hpp:214-278,
tensor_train.hpp:157-191); the run-report CSV keeps report.hpp's schema.
CPU only."""
import os
import subprocess

import numpy as np
import pytest

from oracle.oracle import padded_stride

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.fixture(scope="module")
def rw():
    from oracle.oracle import LIBS, RefWire
    if not os.path.exists(LIBS["reference"]):
        pytest.skip("oracle/_ref not built")
    return RefWire()


def random_tt(rng, dims, ranks):
    from paper_2102_00104_b200.ttsvd import TensorTrain, TTCore
    tt = TensorTrain()
    for j, n in enumerate(dims):
        tt.cores.append(TTCore(np.asfortranarray(rng.standard_normal((ranks[j], n, ranks[j + 1])))))
    return tt


def test_tt_files_cross_read(rw, tmp_path):
    from paper_2102_00104_b200 import wire
    rng = np.random.default_rng(7)
    tt = random_tt(rng, [3, 4, 2, 5], [1, 2, 6, 3, 1])
    p_ours, p_ref = str(tmp_path / "ours.tt"), str(tmp_path / "ref.tt")
    wire.save_tt(tt, p_ours)
    rw.save_tt(p_ref, [c.data for c in tt.cores])
    assert open(p_ours, "rb").read() == open(p_ref, "rb").read()
    back_ref = rw.load_tt(p_ours)
    back_ours = wire.load_tt(p_ref)
    for a, b, c in zip(tt.cores, back_ref, back_ours.cores):
        assert np.array_equal(a.data, b) and np.array_equal(a.data, c.data)
    assert back_ours.ranks() == [1, 2, 6, 3, 1]


def test_tensor_files_cross_read(rw, tmp_path):
    from paper_2102_00104_b200 import wire
    rng = np.random.default_rng(8)
    dims = [5, 7, 3, 4]
    rows = 5 * 7 * 3
    ld = padded_stride(rows)
    X = np.zeros((ld, dims[-1]), order="F")
    X[:rows] = rng.standard_normal((rows, dims[-1]))
    p_ours, p_ref = str(tmp_path / "ours.bin"), str(tmp_path / "ref.bin")
    wire.dump_tensor(X, dims, p_ours)
    rw.dump_tensor(p_ref, X, dims, ld)
    assert open(p_ours, "rb").read() == open(p_ref, "rb").read()
    Y, d2 = rw.load_tensor(p_ours)
    Z, d3 = wire.load_tensor(p_ref)
    assert d2 == dims == d3
    assert np.array_equal(Y[:rows], X[:rows]) and np.array_equal(Z, X)


def test_cpp_header_files_read_by_reference(rw, tmp_path):
    lib = os.path.join(ROOT, "paper_2102_00104_b200")
    exe = str(tmp_path / "dropin")
    r = subprocess.run(["g++", "-std=c++20", "-Wall", "-Werror", f"-I{ROOT}/include", "-I/usr/local/cuda/include",
                        os.path.join(ROOT, "examples", "dropin_example.cpp"), "-o", exe, f"-L{lib}", "-lttsvd_cu",
                        f"-Wl,-rpath,{lib}", "-L/usr/local/cuda/lib64", "-lcudart", "-Wl,-rpath,/usr/local/cuda/lib64"],
                       capture_output=True, text=True)
    assert r.returncode == 0, r.stderr
    r = subprocess.run([exe, "host", str(tmp_path)], capture_output=True, text=True)
    assert r.returncode == 0, (r.returncode, r.stdout, r.stderr)
    X, dims = rw.load_tensor(str(tmp_path / "cpp_tensor.bin"))
    assert dims == [3, 5, 4]
    flat = np.concatenate([X[:15, j] for j in range(4)])
    assert np.array_equal(flat, 0.25 * np.arange(60) - 3.0)
    cores = rw.load_tt(str(tmp_path / "cpp_tt.bin"))
    assert [c.shape for c in cores] == [(1, 3, 2), (2, 5, 3), (3, 4, 1)]
    for j, c in enumerate(cores):
        assert np.array_equal(c.reshape(-1, order="F"), 0.5 * np.arange(c.size) - j)


def test_wire_errors(tmp_path):
    from paper_2102_00104_b200 import wire
    from paper_2102_00104_b200.ttsvd import IoError
    with pytest.raises(IoError):
        wire.load_tt(str(tmp_path / "missing"))
    bad = tmp_path / "bad.bin"
    bad.write_bytes(np.array([2, 3, 4, 999], dtype="<u8").tobytes())  # stride != padded_stride(3)
    with pytest.raises(IoError, match="stride mismatch"):
        wire.load_tensor(str(bad))
    bad.write_bytes(np.array([0], dtype="<u8").tobytes())
    with pytest.raises(IoError, match="bad header"):
        wire.load_tt(str(bad))
    short = tmp_path / "short.tt"
    short.write_bytes(np.array([1, 1, 1, 4], dtype="<u8").tobytes() + b"\0" * 8)
    with pytest.raises(IoError):
        wire.load_tt(str(short))


def test_report_csv_schema_round_trip():
    from paper_2102_00104_b200 import wire
    from paper_2102_00104_b200.ttsvd import StepRecord, TensorTrain
    tt = TensorTrain()
    tt.steps = [StepRecord(1, 1 << 24, 16, 16, 16, 1.0, 1.5e-3, 2e-4, 1.1e-3),
                StepRecord(2, 1 << 20, 256, 32, 256, 0.125, 1.4e-2, 1.6e-3, 1.0e-3)]
    rows = wire.report_rows(tt, "plain", "16^7", 32, 0.0)
    assert [r["phase"] for r in rows[:4]] == ["tsqr", "small-svd", "tsmm", "reorder"]
    assert rows[4]["flops"] == 2 * (1 << 20) * 256 * 256 and rows[6]["bytes"] == 8 * (1 << 20) * (256 + 32)
    text = wire.emit_csv(rows)
    assert text.splitlines()[0] == wire.REPORT_HEADER
    assert wire.parse_csv(text) == rows
    ref_hdr = "/root/reference/proj/include/ttsvd/report.hpp"
    if os.path.exists(ref_hdr):
        assert f'kReportHeader = "{wire.REPORT_HEADER}"' in open(ref_hdr).read()
