"""pytest plugin: run the reference's OWN test suites with the B200 backend
injected through the reference's plugin seam (test harness only).

Loaded with ``-p refsuite_plugin`` by tests/test_gpu_reference_suites.py on
the unmodified reference installed in baseline/_ref (baseline/install_ref.sh).

WG_REFSUITE_TIER=1 -- kernel protocol.  The reference resolves backends by
name from ``kernels._BACKENDS`` and by default from ``kernels.DEFAULT``
(kernels.py:128-163).  Both the "native" entry and the default become one
``B200Backend``: every test that compares "python" against "native"
(test_kernels_backends.py:24-112) then compares the reference's numpy kernels
against the sm_100a kernels bit for bit, and every default-backend call of the
stock engine (test_engine.py, test_acceptance.py) runs its transform / pulls on
the GPU.

WG_REFSUITE_TIER=2 -- whole loop.  ``wedgegraph.run_until_convergence``
(engine.py:330-388) is replaced by the B200 device loop for min-plus programs
(``B200Backend.run_until_convergence``), with the result converted into the
reference's own ``RunResult`` / ``IterationStats`` types; programs without a
kernel descriptor (the generic-path tests, test_engine.py:43-45) and explicit
non-default backends keep the reference loop.
"""

from __future__ import annotations

import os
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent
if str(ROOT) not in sys.path:
    sys.path.insert(0, str(ROOT))

TIER = os.environ.get("WG_REFSUITE_TIER", "1")


def _install():
    import wedgegraph
    import wedgegraph.engine as ref_engine
    import wedgegraph.kernels as ref_kernels

    from paper_1903_07754_b200.backend import B200Backend

    b200 = B200Backend()
    assert "b200.so" not in str(getattr(ref_kernels, "_native", "")), "reference native module shadowed"
    if TIER == "1":
        ref_kernels._BACKENDS["native"] = b200
        ref_kernels.DEFAULT = b200
        return

    stock = ref_engine.run_until_convergence

    def run_until_convergence(topology, index, program, degrees, config, backend=None,
                              frontier_log=None, value_log=None):
        if program.kernel is None or backend not in (None, "auto"):
            return stock(topology, index, program, degrees, config, backend=backend,
                         frontier_log=frontier_log, value_log=value_log)
        n = topology.vertex_count
        if index.vertex_count != n or index.vector_count != topology.vector_count:
            raise ValueError("edge index does not match topology")
        ref_engine._check_weights(topology, program)
        res = b200.run_until_convergence(topology, index, program, degrees, config,
                                         frontier_log=frontier_log, value_log=value_log)
        stats = [ref_engine.IterationStats(
            mode=s.mode, pull_time=s.pull_time, vectors_touched=s.vectors_touched,
            frontier_out_size=s.frontier_out_size, iteration=s.iteration,
            transform_time=s.transform_time, active_edges=s.active_edges,
            active_edge_fraction=s.active_edge_fraction, covered_vectors=s.covered_vectors,
            transform_entries=s.transform_entries) for s in res.stats]
        return ref_engine.RunResult(values=res.values, stats=stats, converged=res.converged)

    ref_engine.run_until_convergence = run_until_convergence
    wedgegraph.run_until_convergence = run_until_convergence


_install()
