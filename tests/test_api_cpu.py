"""Host-side API behaviour that needs no GPU: no CPU fallback, error mapping,
SPEC-type adapters."""

from __future__ import annotations

import numpy as np
import pytest
import torch

from paper_2411_17660_b200 import _lib, dba
from paper_2411_17660_b200.errors import (CalibrationDegenerateError, CapacityError, ConfigError,
                                          FlowSplatError, NumericalError, SolverFailure)


@pytest.mark.skipif(torch.cuda.is_available(), reason="checks the no-GPU behaviour")
def test_no_cpu_fallback():
    with pytest.raises(RuntimeError, match="CUDA device is required"):
        dba.DBASolver(np.array([0]), np.array([1]), 2, 8, 8, (0,))


def test_status_mapping():
    cases = {_lib.DBA_EINVAL: ConfigError, _lib.DBA_ECAPACITY: CapacityError,
             _lib.DBA_ENONFINITE: NumericalError, _lib.DBA_ESOLVER: SolverFailure,
             _lib.DBA_ECALIB: CalibrationDegenerateError}
    for code, exc in cases.items():
        with pytest.raises(exc):
            dba._raise_for(code)
        assert issubclass(exc, FlowSplatError)
    rep = _lib.Report()
    rep.bad_edge = 17
    with pytest.raises(NumericalError) as ei:
        dba._raise_for(_lib.DBA_ENONFINITE, rep)
    assert ei.value.edge == 17
    dba._raise_for(_lib.DBA_OK)


def test_pack_flow_and_state_from_spec_types(reference_flowsplat):
    geometry, providers = reference_flowsplat
    spec = providers.SceneSpec(trajectory="line", frames=4, height=12, width=16)
    sc = providers.SyntheticScene(spec)
    prov = providers.SyntheticProviders(sc)
    edges = [(0, 1), (1, 0), (1, 2)]
    ups = [prov.provide_correspondences(i, j) for i, j in edges]
    prob = dba.BAProblem(edges=edges, updates=ups, fixed=(0,))
    fl = dba._pack_flow(prob, 12, 16)
    assert fl.shape == (3, 12, 16, 4)
    assert np.allclose(fl[1, ..., :2], ups[1].target.astype(np.float32))
    st = dba.BAState([sc.pose_w2c(k) for k in range(4)], np.stack([sc.disparity(k) for k in range(4)]),
                     sc.intrinsics)
    poses, disps, intr = dba._pack_state(st)
    assert poses.shape == (4, 7) and np.allclose(intr, sc.intrinsics.as_vector())
