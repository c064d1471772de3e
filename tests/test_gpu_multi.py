"""Multi-GPU plumbing exercised on one B200 (SURVEY §8 e).

* per-partition generation of configs 4 and 5: partition p of P holds the
  global entries l = p + P * l_local (ttsvd_bench.cpp:72-86), so every P
  builds the same global tensor (noise / uniform parts bit-identical, the
  exact-TT part to rounding);
* the library's own NCCL exchange: tt_svd_distributed_devices (one process,
  ncclCommInitAll, one host thread per device) and a torch.distributed rank
  with an attached communicator (ncclAllGather inside the library) give the
  in-process Alg. 5 result bitwise.  On one GPU the communicator has one rank,
  so the all-gather is a copy; the protocol across ranks is covered by the
  gloo tests (tests/test_distributed_gloo.py).
"""
import os
import subprocess
import sys

import numpy as np
import pytest

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def flat_of(X, dims):
    rows = int(np.prod(dims)) // dims[-1]
    return X[:rows].t().reshape(-1).cpu().numpy()  # Fortran flat order


@pytest.mark.parametrize("P", [2, 4, 8])
def test_config4_partitions_rebuild_the_global_tensor(P):
    from paper_2102_00104_b200 import inputs
    d = 14
    X, dims, _, _ = inputs.config4_slab(1, 0, d)
    g = flat_of(X, dims)
    scale = np.max(np.abs(g))
    for p in range(P):
        Xp, ldims, r_max, eps = inputs.config4_slab(P, p, d)
        assert ldims == [2] * (d - (P.bit_length() - 1)) and r_max == 64
        loc = flat_of(Xp, ldims)
        assert np.max(np.abs(loc - g[p::P])) <= 1e-12 * scale


@pytest.mark.parametrize("P", [2, 4, 8])
def test_config5_partitions_rebuild_the_global_tensor(P):
    import torch
    from paper_2102_00104_b200 import inputs
    d = 5
    X, dims, _, _ = inputs.config5_slab(1, 0, d)
    g = flat_of(X, dims)
    # ||E||^2 over all partitions, the all-reduce of a distributed run
    slabs_e2 = []
    for p in range(P):
        import paper_2102_00104_b200 as tt
        ld = [8 // P] + [8] * (d - 1) if P < 8 else [8] * (d - 1)
        rows = int(np.prod(ld)) // ld[-1]
        E = tt.fortran_empty(rows, ld[-1], ld=tt.padded_stride(rows), zero=True)
        tt.gen_partition(5, 0, E, int(np.prod(ld)), P, p)
        slabs_e2.append(float(torch.sum(E[:rows] ** 2)))
    tot = sum(slabs_e2)
    for p in range(P):
        Xp, ldims, r_max, eps = inputs.config5_slab(P, p, d, allreduce=lambda x: tot)
        loc = flat_of(Xp, ldims)
        assert np.max(np.abs(loc - g[p::P])) <= 1e-11 * np.max(np.abs(g))


def _slabs(P=4, d=10):
    from paper_2102_00104_b200 import inputs
    return [inputs.config4_slab(P, p, d)[0] for p in range(P)], [2] * (d - (P.bit_length() - 1))


def test_devices_driver_matches_in_process_bitwise():
    import paper_2102_00104_b200 as tt
    slabs, ldims = _slabs()
    spec = tt.TruncationSpec(r_max=16)
    a = tt.tt_svd_distributed(slabs, ldims, spec)
    b = tt.tt_svd_distributed_devices([slabs], ldims, spec)
    assert a.ranks() == b.ranks()
    for ca, cb in zip(a.cores, b.cores):
        assert np.array_equal(ca.data, cb.data)


def test_attached_nccl_communicator_matches_in_process(tmp_path):
    script = tmp_path / "rank.py"
    script.write_text(f"""
import os, sys, numpy as np, torch, torch.distributed as dist
sys.path.insert(0, {ROOT!r})
import paper_2102_00104_b200 as tt
from paper_2102_00104_b200 import inputs
os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(29611), RANK="0", WORLD_SIZE="1")
torch.cuda.set_device(0)
dist.init_process_group("nccl", device_id=torch.device("cuda", 0))
slabs = [inputs.config4_slab(2, p, 10)[0] for p in range(2)]
spec = tt.TruncationSpec(r_max=16)
a = tt.tt_svd_distributed(slabs, [2] * 9, spec)
tt.context(0).attach_nccl(dist.group.WORLD)
b = tt.tt_svd_distributed(slabs, [2] * 9, spec, group=dist.group.WORLD, P_total=2, part0=0)
assert a.ranks() == b.ranks(), (a.ranks(), b.ranks())
assert all(np.array_equal(x.data, y.data) for x, y in zip(a.cores, b.cores))
dist.destroy_process_group()
print("nccl ok")
""")
    r = subprocess.run([sys.executable, str(script)], capture_output=True, text=True, timeout=300)
    assert r.returncode == 0 and "nccl ok" in r.stdout, (r.stdout[-2000:], r.stderr[-3000:])
