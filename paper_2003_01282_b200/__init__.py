"""B200-native stochastic Lanczos quadrature (SLQ) engine for spectral graph signatures.

Drop-in for the SLQ hot path of the reference package ``spectrace``
(``/root/reference/pkg/src/spectrace``): ``netlsd_slq``, ``vnge_slq``,
``slq_trace``/``slq_trace_grid`` on graph operators, plus the wave trace.
The compute runs in ``libslq_b200.so`` (hand-written sm_100a CUDA behind a
C ABI declared in ``include/slq_b200.h``); there is no CPU fallback.
"""
from .errors import ConvergenceError, EdgeListError, SlqLibraryError, TridiagonalEigenError
from .graphs import Graph, block_diagonal, csr_from_edges, graph_from_scipy

__version__ = "0.1.0"

_LAZY = {
    # operators.py mirror
    "OperatorKind": "operators", "LinearOperator": "operators", "make_operator": "operators",
    "degrees": "operators", "trace": "operators", "trace_squared": "operators",
    # lanczos.py mirror
    "Tridiagonal": "lanczos", "QuadratureRule": "lanczos", "quadrature_rule": "lanczos",
    "lanczos_tridiagonalize": "lanczos", "extremal_eigenvalues": "lanczos", "dense_spectrum": "lanczos",
    # slq.py mirror
    "SlqConfig": "slq", "SlqEstimate": "slq", "slq_trace": "slq", "slq_trace_grid": "slq",
    "slq_rules": "slq",
    # descriptors.py mirror
    "TimeGrid": "descriptors", "HeatTraceDescriptor": "descriptors", "EntropyValue": "descriptors",
    "WaveTraceDescriptor": "descriptors", "netlsd_slq": "descriptors", "vnge_slq": "descriptors",
    "netlsd_wave_slq": "descriptors", "netlsd_heat_wave_slq": "descriptors",
    "netlsd_slq_sparse": "descriptors", "vnge_slq_sparse": "descriptors",
    "netlsd_taylor": "descriptors", "netlsd_linear": "descriptors", "netlsd_exact": "descriptors",
    "vnge_taylor": "descriptors", "vnge_finger": "descriptors", "vnge_exact": "descriptors",
    "relative_error": "descriptors", "descriptor_distance": "descriptors",
    "descriptor_to_json": "descriptors", "descriptor_from_json": "descriptors",
    # batched small graphs
    "netlsd_slq_batch": "batched", "vnge_slq_batch": "batched", "BatchedGraphs": "batched",
}


def __getattr__(name):
    mod = _LAZY.get(name)
    if mod is None:
        raise AttributeError(name)
    import importlib

    return getattr(importlib.import_module(f".{mod}", __name__), name)
