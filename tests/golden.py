"""Loaders for the committed golden fixtures (made by tests/golden/make_golden.py)."""
import os

import numpy as np

from paper_2003_01282_b200.graphs import Graph

GOLDEN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")


def load(name):
    return np.load(os.path.join(GOLDEN, name), allow_pickle=False)


def graph(z, prefix=""):
    return Graph(n=int(z[f"{prefix}n"]), row_offsets=np.array(z[f"{prefix}offsets"], dtype=np.int64),
                 col_indices=np.array(z[f"{prefix}cols"], dtype=np.int64),
                 weights=np.array(z[f"{prefix}weights"], dtype=np.float64), m=int(z[f"{prefix}m"]))


def rel_l2(a, b):
    a = np.asarray(a, dtype=np.complex128 if np.iscomplexobj(a) or np.iscomplexobj(b) else np.float64)
    b = np.asarray(b, dtype=a.dtype)
    nb = np.linalg.norm(b)
    return float(np.linalg.norm(a - b) / nb) if nb else float(np.linalg.norm(a - b))


def max_rel(a, b, floor=1e-300):
    a = np.asarray(a)
    b = np.asarray(b)
    return float(np.max(np.abs(a - b) / np.maximum(np.abs(b), floor)))
