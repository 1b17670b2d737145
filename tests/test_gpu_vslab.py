"""N2 on one GPU: the velocity-slab decomposition (paper_1204_3853_b200.vslab) emulated with all
slabs in one process (LocalComm: the all-reduce of the slab moments and the halo exchange of the
two boundary velocity columns as device copies), against the oracle and against the undivided GPU
run.  The NCCL transport (DistComm) is the same sequence with torch.distributed collectives; its
neighbour / reduction logic is covered on CPU by tests/test_multirank_cpu.py."""
import numpy as np
import pytest

import inputs
from oracle import scheme, uniform

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu
if not torch.cuda.is_available():
    pytest.skip("no CUDA device", allow_module_level=True)

from paper_1204_3853_b200 import _lib, api  # noqa: E402
from paper_1204_3853_b200.solver import UniformVlasov1D  # noqa: E402
from paper_1204_3853_b200.vslab import LocalComm, VSlabVlasov1D, slab_ranges  # noqa: E402


def _slab_run(w, nslabs, nsteps, recon=scheme.CENTERED4):
    h = inputs.spacing(w)
    G = VSlabVlasov1D(w.ncells, w.lower, h, inputs.background_profile(w), nslabs, range(nslabs), LocalComm(),
                      recon=RECON[recon])
    f0 = inputs.initial_cell_averages(w)
    G.set_state(f0)
    dt = inputs.fixed_dt(w)
    for _ in range(nsteps):
        G.step(dt)
    return np.concatenate(G.get_state(), axis=1), f0, dt


RECON = {scheme.CENTERED4: _lib.CENTERED4, scheme.UPWIND: _lib.UPWIND}


def relerr(a, b):
    return np.max(np.abs(a - b)) / np.max(np.abs(b))


@pytest.mark.parametrize("nslabs", [2, 4])
def test_c1_slabs_match_oracle(nslabs):
    w = inputs.get("C1")
    got, f0, dt = _slab_run(w, nslabs, 1)
    ref, _ = uniform.problem_for(w).run(f0, dt, 1)
    assert relerr(got, ref) < 1e-12
    got, f0, dt = _slab_run(w, nslabs, 50)
    ref, _ = uniform.problem_for(w).run(f0, dt, 50)
    assert relerr(got, ref) < 1e-10


def test_upwind_slabs_match_oracle():
    """UPWIND reconstruction (data-dependent face weights) across the slab faces: the halo carries
    the two neighbour columns its stencils read."""
    w = inputs.get("C1")
    got, f0, dt = _slab_run(w, 2, 10, scheme.UPWIND)
    ref, _ = uniform.problem_for(w, scheme.UPWIND).run(f0, dt, 10)
    assert relerr(got, ref) < 1e-11


def test_c2_four_slabs_hundred_steps():
    w = inputs.get("C2")
    got, f0, dt = _slab_run(w, 4, 100)
    ref, _ = uniform.problem_for(w).run(f0, dt, 100)
    assert relerr(got, ref) < 1e-10


def test_slabs_equal_undivided_gpu_run():
    """Same discretisation, only the moment's summation order and the ghost source differ."""
    w = inputs.scaled(inputs.get("C4"), (128, 1024), (128, 1024))
    got, f0, dt = _slab_run(w, 4, 5)
    S = UniformVlasov1D(w.ncells, w.lower, inputs.spacing(w), inputs.level0_boxes(w), inputs.background_profile(w))
    S.set_state(f0)
    for _ in range(5):
        S.step(dt)
    assert relerr(got, S.get_state()) < 1e-13


def test_pack_unpack_columns():
    w = inputs.scaled(inputs.get("C1"), (16, 32), (16, 32))
    L = api.Level(2, w.ncells, w.lower, inputs.spacing(w), (1, 1), inputs.level0_boxes(w))
    f = L.field(0.0)
    data = np.arange(16 * 32, dtype=np.float64).reshape(16, 32)
    L.set_domain(f, data)
    lo = torch.zeros(32, dtype=torch.float64, device="cuda")
    hi = torch.zeros(32, dtype=torch.float64, device="cuda")
    api.vlasov_vslab_pack(L.h, f, lo, hi)
    torch.cuda.synchronize()
    np.testing.assert_array_equal(lo.cpu().numpy().reshape(16, 2), data[:, 0:2])
    np.testing.assert_array_equal(hi.cpu().numpy().reshape(16, 2), data[:, 30:32])
    api.vlasov_vslab_unpack(L.h, f, hi, lo)             # ghosts: low <- hi columns, high <- lo columns
    torch.cuda.synchronize()
    g = L.patch_view(f, 0, 2).cpu().numpy()[2:-2]
    np.testing.assert_array_equal(g[:, 0:2], data[:, 30:32])
    np.testing.assert_array_equal(g[:, 34:36], data[:, 0:2])
    np.testing.assert_array_equal(g[:, 2:34], data)


def test_slab_ranges():
    assert [len(r) for r in slab_ranges(64, 4)] == [16] * 4
    with pytest.raises(ValueError):
        slab_ranges(64, 3)


_NCCL_SCRIPT = r"""
import os, sys, socket, numpy as np, torch, torch.distributed as dist
sys.path.insert(0, {root!r})
import inputs
from paper_1204_3853_b200.vslab import DistComm, LocalComm, VSlabVlasov1D
s = socket.socket(); s.bind(("127.0.0.1", 0)); port = s.getsockname()[1]; s.close()
os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK="0", WORLD_SIZE="1")
torch.cuda.set_device(0)
dist.init_process_group("nccl", device_id=torch.device("cuda", 0))
w = inputs.scaled(inputs.get("C4"), (256, 512), (64, 64))
h = inputs.spacing(w); dt = inputs.fixed_dt(w)
out = []
for comm in (DistComm.with_p2p_group(0, 1), LocalComm()):
    G = VSlabVlasov1D(w.ncells, w.lower, h, inputs.background_profile(w), 1, [0], comm)
    G.set_state(inputs.initial_cell_averages(w))
    if isinstance(comm, DistComm):
        G.capture(dt)                       # NCCL all-reduce captured in the step graph
        for _ in range(2):
            G.replay()
    else:
        for _ in range(3):
            G.step(dt)
    torch.cuda.synchronize()
    out.append(G.get_state()[0])
np.save({out!r}, np.stack(out))
dist.destroy_process_group()
"""


def test_distcomm_nccl_graph_single_rank(tmp_path):
    """The NCCL transport itself (DistComm: all-reduce on one communicator, halo on a second) in a
    one-rank NCCL process group, with the step captured in a CUDA graph: bitwise the LocalComm run
    (one slab: the all-reduce is the identity and there are no neighbours).  Multi-rank logic:
    tests/test_multirank_cpu.py (gloo, 2 and 3 ranks)."""
    import os
    import subprocess
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    out = str(tmp_path / "o.npy")
    r = subprocess.run([sys.executable, "-c", _NCCL_SCRIPT.format(root=root, out=out)], capture_output=True,
                       text=True, timeout=600)
    assert r.returncode == 0, r.stderr[-3000:]
    a, b = np.load(out)
    np.testing.assert_array_equal(a, b)
