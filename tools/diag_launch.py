"""Host submit time vs device time of one Lanczos run (diagnoses launch-bound behaviour)."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

from paper_2003_01282_b200 import synth
from paper_2003_01282_b200.device import DeviceGraph

g = synth.sbm(100_000, 10, 1e-3, 1e-5, seed=0)
dg = DeviceGraph(g, torch.device("cuda", 0))
for rep in range(4):
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    t0 = time.perf_counter()
    e0.record()
    dg.tridiagonals("normalized_laplacian", 0, 0, 100, 15)
    t1 = time.perf_counter()
    e1.record()
    torch.cuda.synchronize()
    t2 = time.perf_counter()
    print(f"rep {rep}: host submit {1e3 * (t1 - t0):.2f} ms, wall {1e3 * (t2 - t0):.2f} ms, "
          f"device {e0.elapsed_time(e1):.2f} ms")
