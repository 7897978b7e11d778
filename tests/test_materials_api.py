"""Material ABI on the host (no GPU): the fe2_material_t layout of all four
reference material kinds (materials.hpp:37-76) and validation (:80-98)."""
import ctypes as C

import numpy as np
import pytest

import paper_2306_02687_b200 as F
from paper_2306_02687_b200.hrom import _Material


def test_struct_layout():
    assert C.sizeof(_Material) == 8 + 6 * 8
    c = F.CreepParams(1.0, 0.14, 22.09, 1.06, -0.56, 0.25)._c()
    assert c.kind == 3 and list(c.p) == [1.0, 0.14, 22.09, 1.06, -0.56, 0.25]
    p = F.PowerLawParams(1.01, 0.29, 0.0072, 0.08)._c()
    assert p.kind == 2 and list(p.p)[:4] == [1.01, 0.29, 0.0072, 0.08]


@pytest.mark.parametrize("bad", [F.PowerLawParams(N=1.5), F.PowerLawParams(sigma_y0=0.0), F.CreepParams(m=-1.2),
                                 F.CreepParams(A=0.0), F.CreepParams(nu=0.5)])
def test_invalid_parameters_rejected_before_device(bad):
    with pytest.raises(F.Fe2Error) as e:
        F.update_material_batch(bad, np.zeros((1, 3)))
    assert e.value.code == 1  # config


def test_finite_strain_engine_rejects_iterative_materials_before_device():
    """The small-strain engine carries power law / creep (general_return); the
    finite-strain (Biot) engine is J2-only and says so before touching a device."""
    m = F.HyperRomModel(8, 4, 20, 0)
    with pytest.raises(F.Fe2Error) as e:
        F.HyperRomEngine(m.G4, m.w, m.mat, [F.CreepParams(), F.ElasticParams(10.0, 0.3)], m.volume)
    assert e.value.code == 1
