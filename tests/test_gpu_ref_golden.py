"""The sm_100a engine against outputs of the REFERENCE's own code (tests/golden/ref_*,
made by oracle/make_golden.py from /root/reference compiled against the Eigen shim;
see tests/test_ref_golden.py). This pins the device material point and the device HF
RVE solver to the reference directly, not only through the oracle restatement.

Bars: material point — plastic/elastic branch identical per state, stress 1e-13 and
tangent 1e-12 relative (J2 / elastic; the device forms q_tr from an rsqrt seed + Newton
steps, so the last bit may differ), 1e-11 / 1e-9 for the scalar-Newton power-law and
creep return maps (their iteration stops at a tolerance); HF runs — identical Newton
iteration counts per step, Sigma / C_hom 1e-10 relative (dense Cholesky vs the
reference's sparse LDLᵀ).
"""
import os

import numpy as np
import pytest

import paper_2306_02687_b200 as F
from paper_2306_02687_b200.pod import HfRve

from test_ref_golden import HF_CASES, gold, hf_path

pytestmark = pytest.mark.gpu

PRODUCT_MATS = {
    "j2": F.J2LinearParams(1.0, 0.3, 0.01, 0.016),
    "elastic": F.ElasticParams(10.0, 0.3),
    "powerlaw": F.PowerLawParams(1.0, 0.3, 0.01, 0.1),
    "creep": F.CreepParams(1.0, 0.14, 22.09, 1.06, -0.56, 0.05),
}
TOL = {"j2": (1e-13, 1e-12), "elastic": (1e-13, 1e-12), "powerlaw": (1e-11, 1e-9), "creep": (1e-11, 1e-9)}


@pytest.mark.parametrize("kind", list(PRODUCT_MATS))
def test_device_update_material_matches_reference(kind):
    g = gold(f"mat_{kind}")
    sig, C, so, pl = F.update_material_batch(PRODUCT_MATS[kind], g[:, 0:3], g[:, 3:9])
    ts, tc = TOL[kind]
    ref_pl = g[:, 25] > g[:, 7]
    assert np.array_equal(pl, ref_pl)
    scale_s = np.abs(g[:, 9:12]).max(1, keepdims=True)
    scale_c = np.abs(g[:, 12:21]).max(1, keepdims=True)
    assert (np.abs(sig - g[:, 9:12]) / scale_s).max() < ts
    assert (np.abs(C.reshape(-1, 9) - g[:, 12:21]) / scale_c).max() < tc
    assert np.abs(so[:, :5] - g[:, 21:26]).max() < ts * max(1e-3, np.abs(g[:, 21:26]).max())
    assert np.abs(so[:, 5] - g[:, 26]).max() <= ts * np.abs(g[:, 26]).max() + 1e-18


def test_device_soa_constitutive_update_matches_reference():
    """The HBM-streaming SoA kernel (k_material_soa) on the reference's J2 states."""
    import torch

    g = gold("mat_j2")
    N = g.shape[0]
    dev = torch.device("cuda", 0)
    t = lambda a: torch.from_numpy(np.ascontiguousarray(a)).to(dev)  # noqa: E731
    d_eps, d_hin = t(g[:, 0:3].T), t(g[:, 3:8].T)
    d_sig = torch.empty((3, N), dtype=torch.float64, device=dev)
    d_C6 = torch.empty((6, N), dtype=torch.float64, device=dev)
    d_hout = torch.empty((6, N), dtype=torch.float64, device=dev)
    d_pl = torch.empty(N, dtype=torch.uint8, device=dev)
    F.update_material_soa_device(PRODUCT_MATS["j2"], N, d_eps.data_ptr(), d_hin.data_ptr(), d_sig.data_ptr(),
                                 d_C6.data_ptr(), d_hout.data_ptr(), d_pl.data_ptr(),
                                 torch.cuda.current_stream(dev).cuda_stream)
    torch.cuda.synchronize()
    sig, C6, hout, pl = (x.cpu().numpy() for x in (d_sig, d_C6, d_hout, d_pl))
    assert np.array_equal(pl.astype(bool), g[:, 25] > g[:, 7])
    Cref = g[:, 12:21].reshape(-1, 3, 3)[:, [0, 0, 0, 1, 1, 2], [0, 1, 2, 1, 2, 2]]
    assert np.abs(sig.T - g[:, 9:12]).max() < 1e-13 * np.abs(g[:, 9:12]).max()
    assert np.abs(C6.T - Cref).max() < 1e-12 * np.abs(Cref).max()
    assert np.abs(hout.T[:, :5] - g[:, 21:26]).max() < 1e-15


def _hf_materials(kind, dt):
    inc = F.ElasticParams(10.0, 0.3)
    if kind == "j2":
        return (PRODUCT_MATS["j2"], inc)
    if kind == "powerlaw":
        return (PRODUCT_MATS["powerlaw"], inc)
    return (F.CreepParams(1.0, 0.14, 22.09, 1.06, -0.56, dt), inc)


@pytest.mark.parametrize("case", list(HF_CASES))
def test_device_hf_trajectory_matches_reference_run(case):
    """The device HF RVE solver (fe2_hf_*: element kernel, deterministic gather,
    Cholesky; micro_newton / homogenize / run_trajectory on the host) against the
    reference's own run: identical iteration counts per step including the bisected
    steps, Sigma / C_hom to 1e-10, the x_u snapshot columns and committed history."""
    sub, kind, dt, max_iter = HF_CASES[case]
    g, xu = gold(f"hf_{case}"), gold(f"hf_{case}_xu")
    rve = HfRve(sub, _hf_materials(kind, dt))
    r = rve.trajectory(hf_path(case), F.NewtonOptions(1e-8, max_iter, 4), snapshots=True)
    assert np.array_equal(r["iterations"], g[:, 0].astype(int)), (r["iterations"], g[:, 0])
    assert np.abs(r["sigma"] - g[:, 1:4]).max() < 1e-10 * np.abs(g[:, 1:4]).max()
    assert np.abs(r["C"].reshape(-1, 9) - g[:, 4:13]).max() < 1e-10 * np.abs(g[:, 4:13]).max()
    assert np.abs(r["snapshots"] - xu).max() < 1e-10 * np.abs(xu).max()
