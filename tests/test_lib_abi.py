"""The C-ABI library: loads (no GPU needed), exports every symbol declared in
include/dba_b200.h, and its host-side logic (partition, status strings, plan
validation errors that fire before any device work) behaves."""

from __future__ import annotations

import ctypes
import os
import re

import numpy as np
import pytest

from paper_2411_17660_b200 import _lib

HEADER = os.path.join(os.path.dirname(os.path.dirname(__file__)), "include", "dba_b200.h")


def declared_functions():
    txt = open(HEADER).read()
    txt = re.sub(r"/\*.*?\*/", "", txt, flags=re.S)
    return sorted(set(re.findall(r"\b(dba_[a-z0-9_]+)\s*\(", txt)))


@pytest.fixture(scope="module")
def lib():
    return _lib.load()


def test_exports_every_declared_symbol(lib):
    names = declared_functions()
    assert len(names) >= 15
    raw = ctypes.CDLL(str(_lib.lib_path()))
    for n in names:
        assert hasattr(raw, n), n
    assert set(names) <= set(_lib.EXPORTS)


def test_version_and_status(lib):
    assert lib.dba_version() == 1
    assert _lib.status_string(_lib.DBA_ESOLVER).startswith("reduced system singular")
    assert _lib.status_string(99) == "unknown status"


def _py_partition(ii, n, r):
    w = np.ones(n, dtype=np.int64)
    np.add.at(w, ii, 1)
    pre = np.concatenate([[0], np.cumsum(w)])
    b = [0]
    for k in range(1, r):
        f = int(np.searchsorted(pre * r >= k * pre[-1], True))
        f = int(np.argmax(pre * r >= k * pre[-1]))
        b.append(max(f, b[-1]))
    b.append(n)
    return np.array(b)


@pytest.mark.parametrize("n,radius,ranks", [(8, 2, 2), (300, 5, 8), (25, 3, 4), (7, 1, 3)])
def test_partition_matches_reference_rule(n, radius, ranks):
    from paper_2411_17660_b200 import dba, scenes
    ii, jj = scenes.radius_edges(n, radius)
    got = dba.partition(ii, n, ranks)
    assert np.array_equal(got, _py_partition(ii, n, ranks))
    assert got[0] == 0 and got[-1] == n and np.all(np.diff(got) >= 0)


def test_plan_validation_errors(lib):
    """dba_plan_create rejects malformed graphs before touching the device."""
    def create(ii, jj, fixed, n=4):
        ii = np.ascontiguousarray(ii, np.int32)
        jj = np.ascontiguousarray(jj, np.int32)
        fx = np.ascontiguousarray(fixed, np.uint8)
        d = _lib.ProblemDesc(n, 8, 8, len(ii), ii.ctypes.data_as(ctypes.POINTER(ctypes.c_int32)),
                             jj.ctypes.data_as(ctypes.POINTER(ctypes.c_int32)),
                             fx.ctypes.data_as(ctypes.POINTER(ctypes.c_uint8)), 0, 0, -1, 0, 1)
        h = ctypes.c_void_p()
        code = lib.dba_plan_create(ctypes.byref(d), ctypes.byref(h))
        if code == 0:
            lib.dba_plan_destroy(h)
        return code
    assert create([0, 1], [1, 1], [1, 0, 0, 0]) == _lib.DBA_EINVAL      # self edge
    assert create([0, 0], [1, 1], [1, 0, 0, 0]) == _lib.DBA_EINVAL      # duplicate edge
    assert create([0, 5], [1, 2], [1, 0, 0, 0]) == _lib.DBA_EINVAL      # out of range
    assert create([0, 1], [1, 2], [0, 0, 0, 0]) == _lib.DBA_EINVAL      # no gauge anchor
    many = list(range(1, 20))
    assert create([0] * 19, many, [1] + [0] * 19, n=20) == _lib.DBA_ECAPACITY  # out-degree > 16


def test_ctypes_struct_layout_matches_header():
    """Field order/size of the ctypes mirrors vs the C structs (compiled probe)."""
    import subprocess
    import tempfile
    src = r'''
#include <stdio.h>
#include <stddef.h>
#include "dba_b200.h"
int main(void) {
  printf("%zu %zu %zu %zu %zu %zu\n", sizeof(dba_problem_desc), sizeof(dba_options),
         sizeof(dba_buffers), sizeof(dba_report), sizeof(dba_plan_info), sizeof(dba_stats));
  printf("%zu %zu %zu %zu %zu\n", offsetof(dba_report, energy_trace), offsetof(dba_buffers, nccl_comm),
         offsetof(dba_options, calib_cond_max), offsetof(dba_options, damping_candidates),
         offsetof(dba_options, refine));
  return 0;
}'''
    with tempfile.TemporaryDirectory() as d:
        c = os.path.join(d, "probe.c")
        open(c, "w").write(src)
        exe = os.path.join(d, "probe")
        subprocess.run(["gcc", "-I", os.path.dirname(HEADER), c, "-o", exe], check=True)
        out = subprocess.run([exe], capture_output=True, text=True, check=True).stdout.split()
    sizes = [int(x) for x in out]
    assert sizes[:6] == [ctypes.sizeof(t) for t in (_lib.ProblemDesc, _lib.Options, _lib.Buffers,
                                                    _lib.Report, _lib.PlanInfo, _lib.Stats)]
    assert sizes[6] == _lib.Report.energy_trace.offset
    assert sizes[7] == _lib.Buffers.nccl_comm.offset
    assert sizes[8] == _lib.Options.calib_cond_max.offset
    assert sizes[9] == _lib.Options.damping_candidates.offset
    assert sizes[10] == _lib.Options.refine.offset
