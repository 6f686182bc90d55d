"""DSPT ingestion: native reader vs the reference adapter.

CPU tests exercise the host reader of libdba_b200.so (no GPU needed); the GPU test
streams the same files into device memory and solves from them."""

from __future__ import annotations

import struct

import numpy as np
import pytest

from paper_2411_17660_b200 import ingest, scenes
from paper_2411_17660_b200.errors import DataError
from tests.helpers import small_workload


@pytest.fixture(scope="module")
def flow_dir(tmp_path_factory):
    wl = small_workload("C1", height=12, width=16)
    d = tmp_path_factory.mktemp("dspt")
    flow = wl.flow.copy()
    # out-of-range and NaN weights exercise the adapter's clip
    flow[0, 0, 0, 2] = -0.5
    flow[0, 0, 1, 3] = 1.5
    flow[1, 2, 3, 2] = np.nan
    ingest.dump_flows(d, flow, wl.ii, wl.jj)
    prior = np.stack([wl.scene.disparity(k) for k in wl.frames]).astype(np.float32)
    prior[0, 0, 0] = 0.0
    for k in wl.frames:
        scenes.write_dspt(d / ingest.prior_name(k), prior[k])
    return d, wl, flow, prior


def _expected(flow):
    w = flow[..., 2:4]
    w = np.where(w < 0, np.float32(0), np.where(w > 1, np.float32(1), w))
    return np.concatenate([flow[..., :2], w], axis=-1).astype(np.float32)


@pytest.mark.parametrize("threads", [1, 3, 0])
def test_read_flows_matches_restatement(flow_dir, threads):
    d, wl, flow, _ = flow_dir
    got = ingest.read_flows(d, wl.ii, wl.jj, 12, 16, threads=threads)
    exp = _expected(flow)
    assert got.dtype == np.float32 and got.shape == flow.shape
    assert np.array_equal(got, exp, equal_nan=True)
    assert got[0, 0, 0, 2] == 0.0 and got[0, 0, 1, 3] == 1.0 and np.isnan(got[1, 2, 3, 2])


def test_read_flows_matches_reference_adapter(flow_dir, reference_flowsplat):
    _, providers = reference_flowsplat
    d, wl, _, _ = flow_dir
    ref = providers.PrecomputedProviders(d)
    got = ingest.read_flows(d, wl.ii, wl.jj, 12, 16)
    for e, (i, j) in enumerate(zip(wl.ii, wl.jj)):
        upd = ref.provide_correspondences(int(i), int(j))
        exp = np.concatenate([upd.target, upd.weight], axis=-1)
        assert np.array_equal(got[e].astype(np.float64), exp, equal_nan=True)


def test_read_priors_matches_reference_adapter(flow_dir, reference_flowsplat):
    _, providers = reference_flowsplat
    d, wl, _, prior = flow_dir
    got = ingest.read_priors(d, wl.frames, 12, 16)
    assert got[0, 0, 0] == np.float32(1e-6)
    ref = providers.PrecomputedProviders(d)
    for k in wl.frames:
        exp = ref.provide_depth_prior(k)
        # the reference clamps in float64; the float32 payload agrees except at the clamp
        ok = exp > 1e-6
        assert np.array_equal(got[k][ok].astype(np.float64), exp[ok])


def _corrupt(path, how):
    raw = bytearray(path.read_bytes())
    if how == "magic":
        raw[:4] = b"DSPX"
    elif how == "version":
        raw[4:8] = struct.pack("<I", 2)
    elif how == "truncated":
        raw = raw[:-4]
    elif how == "channels":
        raw[16:20] = struct.pack("<I", 3)
    elif how == "shape":
        raw[8:12] = struct.pack("<I", 16)
        raw[12:16] = struct.pack("<I", 12)
    path.write_bytes(bytes(raw))


@pytest.mark.parametrize("how", ["missing", "magic", "version", "truncated", "channels", "shape"])
def test_malformed_files_raise_data_error(tmp_path, how):
    wl = small_workload("C1", height=12, width=16)
    ingest.dump_flows(tmp_path, wl.flow, wl.ii, wl.jj)
    for e in (7, 3):  # the smallest failing index is reported
        p = tmp_path / ingest.flow_name(wl.ii[e], wl.jj[e])
        if how == "missing":
            p.unlink()
        else:
            _corrupt(p, how)
    with pytest.raises(DataError) as ei:
        ingest.read_flows(tmp_path, wl.ii, wl.jj, 12, 16)
    assert ingest.flow_name(wl.ii[3], wl.jj[3]) in str(ei.value)
    assert "(index 3)" in str(ei.value)


def test_empty_edge_list(tmp_path):
    out = ingest.read_flows(tmp_path, [], [], 12, 16)
    assert out.shape == (0, 12, 16, 4)


@pytest.mark.gpu
def test_load_flows_device_and_solve(flow_dir):
    import torch

    from paper_2411_17660_b200 import dba
    d, wl, flow, _ = flow_dir
    host = ingest.read_flows(d, wl.ii, wl.jj, 12, 16)
    # a staging buffer of two records forces one copy per record pair
    dev = ingest.load_flows(d, wl.ii, wl.jj, 12, 16, staging_mb=0)
    assert dev.is_cuda and np.array_equal(dev.cpu().numpy(), host, equal_nan=True)
    clean = small_workload("C1", height=12, width=16)
    ingest.dump_flows(d / "clean", clean.flow, clean.ii, clean.jj)
    fdev = ingest.load_flows(d / "clean", clean.ii, clean.jj, 12, 16)
    s = dba.DBASolver(clean.ii, clean.jj, len(clean.frames), 12, 16, clean.fixed)
    a = s.solve(clean.poses0, clean.disps0, clean.intr0, fdev, iters=2)
    b = s.solve(clean.poses0, clean.disps0, clean.intr0, torch.as_tensor(clean.flow, device="cuda"), iters=2)
    assert torch.equal(a[0], b[0]) and torch.equal(a[1], b[1])
