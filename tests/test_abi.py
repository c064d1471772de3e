"""CPU checks of the drop-in boundary: the C-ABI library loads, exports every
symbol include/ttsvd_cu.h declares, and fails cleanly (status code, message)
without a GPU.  No compute calls here."""
import ctypes as C
import os

import numpy as np
import pytest


def test_library_exports_every_header_symbol():
    from paper_2102_00104_b200 import _lib
    L = _lib.lib()
    syms = _lib.header_symbols()
    assert len(syms) >= 25
    missing = [s for s in syms if not hasattr(L, s)]
    assert not missing, missing
    # and the ctypes signature table covers the header exactly
    assert sorted(_lib._SIGS) == syms


def test_no_gpu_is_a_clean_error():
    import torch
    if torch.cuda.is_available():
        pytest.skip("GPU present")
    from paper_2102_00104_b200 import _lib
    L = _lib.lib()
    h = C.c_void_p()
    rc = L.ttsvd_cu_ctx_create(0, None, C.byref(h))
    assert rc == 8  # TTSVD_ERR_DEVICE
    assert L.ttsvd_cu_last_error()


def test_host_arithmetic_entries():
    from paper_2102_00104_b200 import _lib
    L = _lib.lib()
    # shape.hpp:22-28 pins (test_storage.cpp:11-17)
    for n, s in [(1, 64), (64, 64), (65, 192), (128, 192), (256, 320), (262144, 262208), (1 << 24, (1 << 24) + 64)]:
        assert L.ttsvd_cu_padded_stride(n) == s
    out = C.c_double()
    assert L.ttsvd_cu_derive_delta(2.0, 0.1, 5, C.byref(out)) == 0 and abs(out.value - 0.1) < 1e-15
    assert L.ttsvd_cu_derive_delta(1.0, 0.1, 1, C.byref(out)) == 6


def test_c_header_compiles_standalone(tmp_path):
    src = tmp_path / "t.c"
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    src.write_text('#include "ttsvd_cu.h"\nint main(void){return ttsvd_cu_padded_stride(1)==64?0:1;}\n')
    import subprocess
    lib = os.path.join(root, "paper_2102_00104_b200")
    r = subprocess.run(["gcc", "-std=c99", "-Wall", "-Werror", f"-I{root}/include", str(src), "-o",
                        str(tmp_path / "t"), f"-L{lib}", "-lttsvd_cu", f"-Wl,-rpath,{lib}"],
                       capture_output=True, text=True)
    assert r.returncode == 0, r.stderr
    assert subprocess.run([str(tmp_path / "t")]).returncode == 0


def _build_example(tmp_path):
    import subprocess
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    lib = os.path.join(root, "paper_2102_00104_b200")
    exe = str(tmp_path / "dropin")
    r = subprocess.run(["g++", "-std=c++20", "-Wall", "-Werror", f"-I{root}/include", "-I/usr/local/cuda/include",
                        os.path.join(root, "examples", "dropin_example.cpp"), "-o", exe, f"-L{lib}", "-lttsvd_cu",
                        f"-Wl,-rpath,{lib}", "-L/usr/local/cuda/lib64", "-lcudart", "-Wl,-rpath,/usr/local/cuda/lib64"],
                       capture_output=True, text=True)
    assert r.returncode == 0, r.stderr
    return exe


def test_cpp_dropin_header_compiles_and_host_entries_run(tmp_path):
    """include/ttsvd_b200.hpp: the reference's names/types over the C-ABI."""
    import subprocess
    exe = _build_example(tmp_path)
    r = subprocess.run([exe, "host"], capture_output=True, text=True)
    assert r.returncode == 0, (r.returncode, r.stdout, r.stderr)


@pytest.mark.gpu
def test_cpp_dropin_device_path(tmp_path):
    import subprocess
    exe = _build_example(tmp_path)
    r = subprocess.run([exe], capture_output=True, text=True, timeout=300)
    assert r.returncode == 0, (r.returncode, r.stdout, r.stderr)
    assert "device entry points ok" in r.stdout


@pytest.mark.parametrize("dims,m_min,f1_min,r_tilde,r_max", [
    ([4] * 10, 16, 0.5, (), 16), ([2] * 20, 16, 0.5, (), 64), ([16] * 7, 16, 0.5, (), 32),
    ([3, 5, 7, 2], 64, 0.25, (), 8), ([2] * 8, 4096, 0.5, (), 4), ([5, 6], 2, 1.0, (3,), 10),
    ([2] * 10, 16, 0.5, (2, 4, 8, 16, 32, 16, 8, 4, 2), 100)])
def test_choose_combined_dims_matches_reference(dims, m_min, f1_min, r_tilde, r_max, ref):
    # tt_svd.hpp:316-330 — host arithmetic of the C-ABI, no GPU needed
    import ctypes as C
    from paper_2102_00104_b200 import _lib
    L = _lib.lib()
    dv = np.asarray(dims, dtype=np.int64)
    rt = np.asarray(r_tilde, dtype=np.int64)
    k, m = C.c_int64(), C.c_int64()
    rc = L.ttsvd_cu_choose_combined_dims(dv.ctypes.data_as(_lib.i64p), len(dv), m_min, f1_min,
                                         rt.ctypes.data if len(rt) else None, len(rt), r_max, C.byref(k),
                                         C.byref(m))
    assert rc == 0
    assert (k.value, m.value) == ref.choose_combined_dims(dims, m_min, f1_min, r_tilde, r_max)
