"""GPU synthetic correspondence provider.

``synthetic_flows(scene, ii, jj)`` returns the (E, H, W, 4) float32 flow records of
``SyntheticProviders.provide_correspondences`` (``providers.py:318-338``) for a batch of
edges, computed on the device by ``dba_synthetic_flows`` (``csrc/dba_provider.cu``): one
thread per edge-pixel ray-casts the analytic scene, reprojects through the exact
disparity and tests visibility from the target camera.  Pixel noise, when the scene
has any, is drawn on the host with the reference's seeding (``providers.py:333-335``)
and added to the targets.
"""

from __future__ import annotations

import ctypes

import numpy as np
import torch

from . import _lib
from .dba import _device, _raise_for
from .scenes import OUTER_RADIUS


def synthetic_flows(scene, ii, jj, device=None, stream=None):
    lib = _lib.load()
    dev = _device(device)
    sp = scene.spec
    ii = np.ascontiguousarray(ii, dtype=np.int32)
    jj = np.ascontiguousarray(jj, dtype=np.int32)
    E = len(ii)
    out = torch.empty((E, sp.height, sp.width, 4), dtype=torch.float32, device=dev)
    if E == 0:
        return out
    if min(ii.min(), jj.min()) < 0 or max(ii.max(), jj.max()) >= sp.frames:
        raise ValueError("edge references a frame outside the scene")
    c2w = torch.as_tensor(scene.c2w, dtype=torch.float64, device=dev).contiguous()
    w2c = torch.as_tensor(scene.w2c, dtype=torch.float64, device=dev).contiguous()
    occ = torch.as_tensor(np.concatenate([scene.centers, scene.radii[:, None]], axis=1).reshape(-1, 4),
                          dtype=torch.float64, device=dev).contiguous()
    ti = torch.as_tensor(ii, device=dev)
    tj = torch.as_tensor(jj, device=dev)
    intr = np.ascontiguousarray(scene.intr, dtype=np.float64)
    st = stream if stream is not None else torch.cuda.current_stream(dev)
    with torch.cuda.device(dev):
        _raise_for(lib.dba_synthetic_flows(
            sp.height, sp.width, intr.ctypes.data_as(ctypes.POINTER(ctypes.c_double)), float(OUTER_RADIUS),
            len(scene.radii), ctypes.c_void_p(occ.data_ptr() if len(scene.radii) else 0),
            ctypes.c_void_p(c2w.data_ptr()), ctypes.c_void_p(w2c.data_ptr()), E,
            ctypes.c_void_p(ti.data_ptr()), ctypes.c_void_p(tj.data_ptr()), ctypes.c_void_p(out.data_ptr()),
            ctypes.c_void_p(st.cuda_stream)))
    if sp.pixel_noise > 0:
        noise = np.stack([np.random.default_rng(np.random.SeedSequence([sp.seed, 31, int(i), int(j)])).normal(
            size=(sp.height, sp.width, 2)) for i, j in zip(ii, jj)])
        out[..., :2] += torch.as_tensor(sp.pixel_noise * noise, dtype=torch.float32, device=dev)
    return out
