"""Where does the end-to-end (host Graph -> descriptors) time go?"""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

from paper_2003_01282_b200 import synth
from paper_2003_01282_b200.descriptors import TimeGrid, netlsd_heat_wave_slq
from paper_2003_01282_b200.graphs import Graph
from paper_2003_01282_b200.slq import SlqConfig

g0 = synth.sbm(100_000, 10, 1e-3, 1e-5, seed=0)
pin = [torch.tensor(np.array(a)).pin_memory() for a in (g0.row_offsets, g0.col_indices, g0.weights)]
grid = TimeGrid(1e-2, 1e2, 250)
cfg = SlqConfig(n_v=100, s=15, seed=0)
torch.cuda.synchronize()
for rep in range(6):
    g = Graph(n=g0.n, row_offsets=pin[0].numpy(), col_indices=pin[1].numpy(), weights=pin[2].numpy(), m=g0.m)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    from paper_2003_01282_b200.operators import OperatorKind, make_operator
    op = make_operator(g, OperatorKind.NORMALIZED_LAPLACIAN)
    t1 = time.perf_counter()
    from paper_2003_01282_b200.slq import slq_rules
    rules = slq_rules(op, cfg)
    t2 = time.perf_counter()
    vals, stds = rules.integrate(grid.values, [0, 1, 2])
    t3 = time.perf_counter()
    v = vals.cpu().numpy()
    t4 = time.perf_counter()
    torch.cuda.synchronize()
    g2 = Graph(n=g0.n, row_offsets=pin[0].numpy(), col_indices=pin[1].numpy(), weights=pin[2].numpy(), m=g0.m)
    torch.cuda.synchronize()
    t5 = time.perf_counter()
    heat, wave = netlsd_heat_wave_slq(g2, grid, cfg, with_hash=False)
    t6 = time.perf_counter()
    print(f"make_operator {1e3*(t1-t0):.2f}  rules-submit {1e3*(t2-t1):.2f}  integrate-submit {1e3*(t3-t2):.2f} "
          f"d2h(wait) {1e3*(t4-t3):.2f}  | api total {1e3*(t6-t5):.2f} ms")
