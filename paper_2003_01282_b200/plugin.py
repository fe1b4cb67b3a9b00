"""Reference-side plugin: route the reference's SLQ seam through libslq_b200.so.

The reference (``spectrace``) collects one Gauss rule per probe in
``_collect_rules(op, cfg, threads)`` (``/root/reference/pkg/src/spectrace/slq.py:80-86``);
everything above it (``_apply_rule``, ``_estimate_from``, the descriptor objects) is O(n_v*s*T)
host arithmetic.  ``install(spectrace)`` replaces exactly that seam:

* ``make_operator`` (``operators.py:65-102``) is wrapped so every graph operator it builds is
  remembered together with its ``Graph`` and ``OperatorKind`` (the reference's ``LinearOperator``
  is a closure and does not carry its graph);
* ``_collect_rules`` looks the operator up and runs the whole batched Lanczos + Gauss-rule
  computation on the GPU (``slq_rules_seeded`` through ``paper_2003_01282_b200``), returning the
  reference's own ``QuadratureRule`` objects in probe order.

The reference's host code then integrates, aggregates and builds its descriptors unchanged, so
``spectrace.netlsd_slq`` / ``vnge_slq`` / ``slq_trace_grid`` return the reference's types with
device-computed rules.  Operators the plugin did not see being built (the reference's
``explicit_operator`` test fakes, user closures) are not accelerated: by default they raise
``TypeError`` (there is no CPU path in this package); ``unknown_ops="reference"`` leaves them on the
reference's own unmodified code instead.  ``INTEGRATION.md`` shows the equivalent two-line source
patch a maintainer would commit.
"""
from __future__ import annotations

import sys
import weakref

import numpy as np

__all__ = ["collect_rules", "install", "Installed"]


def collect_rules(graph, kind, cfg, *, dtype: str = "f64") -> list[tuple[np.ndarray, np.ndarray]]:
    """Per-probe ``(nodes, weights)`` of probes 0..cfg.n_v-1 on the GPU: the output of the reference's
    ``_collect_rules`` (``slq.py:80-86``; nodes clipped to the operator interval, ``slq.py:74-77``).

    ``graph``: the reference's ``Graph`` or this package's; ``kind``: an ``OperatorKind`` of either
    package or its string value; ``cfg``: any object with ``n_v``, ``s``, ``distribution``, ``seed``."""
    from .operators import make_operator
    from .slq import slq_rules

    op = make_operator(graph, getattr(kind, "value", kind))
    rules = slq_rules(op, cfg, dtype=dtype)
    rules.check()
    nodes = rules.nodes.cpu().numpy()
    weights = rules.weights.cpu().numpy()
    steps = rules.steps.cpu().numpy()
    return [(nodes[p, :steps[p]].copy(), weights[p, :steps[p]].copy()) for p in range(rules.count)]


class Installed:
    """Handle of an installed plugin; ``uninstall()`` restores the reference's functions."""

    def __init__(self, patches):
        self._patches = patches
        self.gpu_calls = 0

    def uninstall(self) -> None:
        for mod, name, orig in reversed(self._patches):
            setattr(mod, name, orig)
        self._patches = []


def install(spectrace, *, unknown_ops: str = "raise", dtype: str = "f64") -> Installed:
    """Patch an imported ``spectrace`` package so its ``_collect_rules`` seam runs on the GPU."""
    if unknown_ops not in ("raise", "reference"):
        raise ValueError("unknown_ops must be 'raise' or 'reference'")
    ops_mod = sys.modules[spectrace.__name__ + ".operators"]
    slq_mod = sys.modules[spectrace.__name__ + ".slq"]
    lan_mod = sys.modules[spectrace.__name__ + ".lanczos"]
    orig_make = ops_mod.make_operator
    orig_collect = slq_mod._collect_rules
    quad_rule = lan_mod.QuadratureRule
    graphs_of: dict = {}   # id(op) -> (weakref(op), graph, kind)

    def make_operator(g, kind):
        op = orig_make(g, kind)
        key = id(op)
        try:
            ref = weakref.ref(op, lambda _r, key=key: graphs_of.pop(key, None))
        except TypeError:
            ref = (lambda op=op: op)
        graphs_of[key] = (ref, g, kind)
        return op

    handle = None

    def _collect_rules(op, cfg, threads):
        hit = graphs_of.get(id(op))
        if hit is None or hit[0]() is not op:
            if unknown_ops == "reference":
                return orig_collect(op, cfg, threads)
            raise TypeError("paper_2003_01282_b200 plugin: only operators built by make_operator(graph, kind) run "
                            "on the GPU (no CPU fallback); install(..., unknown_ops='reference') keeps others on "
                            "the reference path")
        _, g, kind = hit
        handle.gpu_calls += 1
        return [quad_rule(nodes=n, weights=w) for n, w in collect_rules(g, kind, cfg, dtype=dtype)]

    patches = []
    for name, mod in list(sys.modules.items()):
        if mod is None or not (name == spectrace.__name__ or name.startswith(spectrace.__name__ + ".")):
            continue
        if getattr(mod, "make_operator", None) is orig_make:
            patches.append((mod, "make_operator", orig_make))
            mod.make_operator = make_operator
    patches.append((slq_mod, "_collect_rules", orig_collect))
    slq_mod._collect_rules = _collect_rules
    handle = Installed(patches)
    return handle
