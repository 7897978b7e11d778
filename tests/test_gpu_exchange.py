"""The multi-GPU exchange through the C ABI (fe2_hrom_gather):
device-side packing of {Σ | C | ‖r‖ | status} per point, in-place NCCL
all-gather, max all-reduce of the failure flag. One GPU here, so the
communicator has one rank: the gathered block must equal the rank's own
records bit for bit (the same layout as shard.pack_outputs, which the gloo
tests exercise at world size 2), and the flag must follow the statuses."""
import numpy as np
import pytest
import torch

import paper_2306_02687_b200 as F
from paper_2306_02687_b200.shard import PACK, pack_outputs

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def comm():
    c = F.NcclComm(0, 1, 0, F.nccl_unique_id())
    yield c
    c.close()


def test_gather_small_strain_matches_pack(comm):
    m = F.HyperRomModel(33, 12, 200, 0)
    P = 300
    E = F.make_paths(0, 0, P, 4)
    eng = F.HyperRomEngine.from_model(m)
    eng.alloc_points(P)
    for k in range(4):
        out = eng.solve_increment(E[:, k])
        d_all = torch.full((1, P, PACK), np.nan, dtype=torch.float64, device="cuda:0")
        failed = eng.gather(comm, d_all.data_ptr())  # the handle's own output buffers
        ref = pack_outputs(out["sigma"], out["C"], out["res_norm"], out["status"])
        np.testing.assert_array_equal(d_all[0].cpu().numpy(), ref)
        assert failed is False


def test_gather_explicit_device_buffers_and_failure_flag(comm):
    m = F.HyperRomModel(33, 12, 200, 0)
    P = 256
    E = F.make_paths(0, 0, P, 20)
    eng = F.HyperRomEngine.from_model(m)
    eng.alloc_points(P)
    dev = torch.device("cuda", 0)
    dE = torch.from_numpy(np.ascontiguousarray(E[:, 19])).to(dev)  # one jump to the end of the path
    sig = torch.empty((P, 3), dtype=torch.float64, device=dev)
    Cm = torch.empty((P, 9), dtype=torch.float64, device=dev)
    res = torch.empty(P, dtype=torch.float64, device=dev)
    it, pc, st = (torch.empty(P, dtype=torch.int32, device=dev) for _ in range(3))
    opts = F.NewtonOptions(max_iter=1, max_bisections=0)  # forces solver failures
    eng.solve_increment_device(dE.data_ptr(), sig.data_ptr(), Cm.data_ptr(), it.data_ptr(), pc.data_ptr(),
                               res.data_ptr(), st.data_ptr(), opts=opts)
    torch.cuda.synchronize()
    status = st.cpu().numpy()
    assert (status != 0).any()
    d_all = torch.empty((1, P, PACK), dtype=torch.float64, device=dev)
    failed = eng.gather(comm, d_all.data_ptr(), sig.data_ptr(), Cm.data_ptr(), res.data_ptr(), st.data_ptr())
    assert failed is True
    got = d_all[0].cpu().numpy()
    np.testing.assert_array_equal(got[:, 13], status.astype(np.float64))
    ok = status == 0
    np.testing.assert_array_equal(got[ok, 0:3], sig.cpu().numpy()[ok])
    np.testing.assert_array_equal(got[ok, 3:12], Cm.cpu().numpy()[ok])


def test_gather_finite_strain_record_width(comm):
    m = F.HyperRomModel(33, 8, 120, 1)
    P = 64
    E = F.make_paths(2, 1, P, 3)
    eng = F.HyperRomEngine.from_model(m, finite_strain=True)
    eng.alloc_points(P)
    out = eng.solve_increment(E[:, 2])
    d_all = torch.empty((1, P, 4 + 16 + 2), dtype=torch.float64, device="cuda:0")
    assert eng.gather(comm, d_all.data_ptr()) is False
    got = d_all[0].cpu().numpy()
    np.testing.assert_array_equal(got[:, 0:4], out["sigma"].reshape(P, 4))
    np.testing.assert_array_equal(got[:, 4:20], out["C"].reshape(P, 16))
    np.testing.assert_array_equal(got[:, 20], out["res_norm"])
    np.testing.assert_array_equal(got[:, 21], out["status"])
