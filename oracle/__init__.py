"""CPU oracle for the DBA Gauss-Newton step — TEST INFRASTRUCTURE ONLY.

This package is the checker, never the product.  Only ``tests/``,
``__graft_entry__.smoke()`` and ``bench.py``'s ``cpu_baseline`` / ``--impl
reference`` legs may import it.  The product path (``paper_2411_17660_b200``)
never imports anything from here and fails loudly when its CUDA library is
missing.

Contents
--------
geometry   float64 numpy restatement of ``/root/reference/pkg/src/flowsplat/geometry.py``
           (pinned against the reference's own tests + golden vectors in tests/golden).
dba        float64 restatement of the SPEC's dense bundle adjustment
           (``/root/reference/SPEC.md:286-394``).  The reference ships NO dba
           module (``__init__.py:8`` names it, the file is absent): DBA parity is
           UNPINNED by reference code ("parity unpinned"); it is pinned by the
           SPEC's own properties (finite-difference Jacobians,
           Schur == dense joint solve, zero energy at truth, fixed point at
           truth, monotone energy, 8-keyframe recovery) — see DESIGN.md §Oracle.
sharded    the same algorithm over a frame partition (partial systems summed),
           used to check the multi-rank decomposition on CPU.
"""
