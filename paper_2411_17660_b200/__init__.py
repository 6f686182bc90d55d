"""paper_2411_17660_b200 — B200-native dense bundle adjustment (DROID-Splat DBA step).

The drop-in for the reference's ``flowsplat.dba`` module:
``solve_ba``, ``solve_ba_calib``, ``energy``, ``energy_rgbd`` and the tensor API
``DBASolver`` / ``gn_solve``, all running hand-written sm_100a kernels through the
C-ABI in ``include/dba_b200.h`` (``libdba_b200.so``, built in-tree).
"""

from .errors import (CalibrationDegenerateError, CapacityError, ConfigError, DataError,
                     FlowSplatError, NumericalError, SolverFailure)

__version__ = "0.1.0"

__all__ = [
    "FlowSplatError", "ConfigError", "DataError", "CapacityError", "NumericalError",
    "SolverFailure", "CalibrationDegenerateError",
]


def __getattr__(name):
    # the solver API imports torch + the CUDA library lazily
    if name in ("dba", "scenes", "geometry", "ingest"):
        import importlib
        return importlib.import_module(f".{name}", __name__)
    raise AttributeError(name)
