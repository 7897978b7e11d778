"""The multi-GPU exchange through the C ABI (fe2_hrom_gather):
device-side packing of {Σ | C | ‖r‖ | status} per point, in-place NCCL
all-gather, max all-reduce of the failure and residual flags. With one GPU the
communicator has one rank: the gathered block must equal the rank's own
records bit for bit (the same layout as shard.pack_outputs, which the gloo
tests exercise at world size 2), and the flags must follow the statuses and
residuals. With two or more GPUs, a real two-rank run with unequal blocks is
checked against a single-device run (skipped below 2 GPUs)."""
import os

import numpy as np
import pytest
import torch
import torch.multiprocessing as mp

import paper_2306_02687_b200 as F
from paper_2306_02687_b200.shard import PACK, gather_rows, pack_outputs, shard_range

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


def test_gather_residual_flag_and_async(comm):
    """flags[1] = some point with ||r|| > res_tol (the monolithic lockstep test);
    wait=False leaves the exchange queued on the stream."""
    m = F.HyperRomModel(33, 12, 200, 0)
    P = 128
    E = F.make_paths(0, 0, P, 4)
    eng = F.HyperRomEngine.from_model(m)
    eng.alloc_points(P)
    out = eng.solve_increment(E[:, 3])
    d_all = torch.empty((1, P, PACK), dtype=torch.float64, device="cuda:0")
    assert eng.gather_layout(comm) == (P, [P])
    rmax = float(out["res_norm"].max())
    assert eng.gather(comm, d_all.data_ptr(), res_tol=rmax, flags=True) == (False, False)
    assert eng.gather(comm, d_all.data_ptr(), res_tol=rmax * 0.5, flags=True) == (False, True)
    d_all.zero_()
    assert eng.gather(comm, d_all.data_ptr(), wait=False) is None
    torch.cuda.synchronize()
    np.testing.assert_array_equal(d_all[0].cpu().numpy(),
                                  pack_outputs(out["sigma"], out["C"], out["res_norm"], out["status"]))


def test_mono_iterate_device_equals_host_api():
    """fe2_hrom_mono_iterate_device (device E, asynchronous) gives the host call's outputs bit for bit."""
    m = F.HyperRomModel(33, 12, 200, 0)
    P = 200
    E = F.make_paths(0, 0, P, 6)
    host = F.HyperRomEngine.from_model(m)
    devc = F.HyperRomEngine.from_model(m)
    host.alloc_points(P)
    devc.alloc_points(P)
    p_sig, p_C, _, p_pc, p_res, p_st = devc.output_ptrs()
    dev = torch.device("cuda", 0)
    for k in range(6):
        host.mono_begin()
        devc.mono_begin()
        dE = torch.from_numpy(np.ascontiguousarray(E[:, k])).to(dev)
        for it in range(3):
            a = host.mono_iterate(E[:, k])
            devc.mono_iterate_device(dE.data_ptr())
            torch.cuda.synchronize()
            np.testing.assert_array_equal(_dev_to_np(p_sig, (P, 3), np.float64), a["sigma"])
            np.testing.assert_array_equal(_dev_to_np(p_C, (P, 9), np.float64), a["C"].reshape(P, 9))
            np.testing.assert_array_equal(_dev_to_np(p_res, (P,), np.float64), a["rel_res"])
            np.testing.assert_array_equal(_dev_to_np(p_st, (P,), np.int32), a["status"])
        host.mono_commit()
        devc.mono_commit()


def _dev_to_np(ptr, shape, dtype):
    class _B:
        __cuda_array_interface__ = {"shape": shape, "typestr": np.dtype(dtype).str, "data": (ptr, False),
                                    "version": 3, "strides": None, "stream": None}
    return torch.as_tensor(_B(), device="cuda:0").cpu().numpy()


P2_TOTAL, P2_INCR = 557, 5  # two unequal blocks (279, 278)


def _two_rank_worker(rank, world, uid, out_dir):
    torch.cuda.set_device(rank)
    m = F.HyperRomModel(33, 12, 200, 0)
    p0, p1 = shard_range(P2_TOTAL, rank, world)
    E = F.make_paths(0, 0, p1 - p0, P2_INCR, p0=p0)
    eng = F.HyperRomEngine.from_model(m, device=rank)
    eng.alloc_points(p1 - p0)
    comm = F.NcclComm(rank, world, rank, uid)
    pmax, counts = eng.gather_layout(comm)
    d_all = torch.empty((world, pmax, PACK), dtype=torch.float64, device=f"cuda:{rank}")
    res = []
    for k in range(P2_INCR):
        eng.solve_increment(E[:, k])
        failed = eng.gather(comm, d_all.data_ptr())
        assert failed is False
        res.append(d_all.cpu().numpy())
    np.save(os.path.join(out_dir, f"rank{rank}.npy"), np.stack(res))
    np.save(os.path.join(out_dir, f"counts{rank}.npy"), np.array(counts))
    comm.close()


@pytest.mark.skipif(torch.cuda.device_count() < 2, reason="needs 2 GPUs (one process per GPU)")
def test_two_rank_gather_unequal_blocks_equals_single_device(tmp_path):
    world = 2
    uid = F.nccl_unique_id()
    mp.start_processes(_two_rank_worker, args=(world, uid, str(tmp_path)), nprocs=world, join=True,
                       start_method="spawn")
    counts = np.load(tmp_path / "counts0.npy").tolist()
    assert counts == [279, 278]
    g0, g1 = np.load(tmp_path / "rank0.npy"), np.load(tmp_path / "rank1.npy")
    np.testing.assert_array_equal(g0, g1)  # every rank holds the same gathered records
    m = F.HyperRomModel(33, 12, 200, 0)
    E = F.make_paths(0, 0, P2_TOTAL, P2_INCR)
    eng = F.HyperRomEngine.from_model(m)
    eng.alloc_points(P2_TOTAL)
    rows = gather_rows(counts)
    for k in range(P2_INCR):
        out = eng.solve_increment(E[:, k])
        flat = g0[k].reshape(-1, PACK)
        np.testing.assert_array_equal(flat[rows], pack_outputs(out["sigma"], out["C"], out["res_norm"], out["status"]))
        pad = np.setdiff1d(np.arange(flat.shape[0]), rows)
        assert (flat[pad, 13] == -1).all()
