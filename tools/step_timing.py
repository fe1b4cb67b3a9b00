"""Per-phase device time of the CGS step kernels (SLQ_STEP_TIMING=1): CTA 0 stamps %globaltimer at
kernel start and around every grid barrier; prints, per step, the work before each barrier and the
wait inside it (the wait includes the slowest CTA).  C2 workload (SBM-100k, 100 fp64 probes)."""
import ctypes
import os
import sys

os.environ["SLQ_STEP_TIMING"] = "1"
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

from paper_2003_01282_b200 import _lib, synth
from paper_2003_01282_b200.device import DeviceGraph

dev = torch.device("cuda", 0)
dg = DeviceGraph(synth.sbm(100_000, 10, 1e-3, 1e-5, seed=0), dev)
for _ in range(3):
    dg.rules("normalized_laplacian", 0, 0, 100, 15).check()
torch.cuda.synchronize()
lib = _lib.load()
buf = (ctypes.c_ulonglong * (32 * 128))()
lib.slq_debug_step_times.restype = ctypes.c_int
n = lib.slq_debug_step_times(buf, 32 * 128)
t = np.array(buf[:n], dtype=np.float64).reshape(128, 32)
for i in range(14):
    row = t[i]
    k = [j for j in range(32) if row[j] > 0]
    stamps = row[:max(k) + 1] - row[0]
    work = [stamps[2 * b + 1] - stamps[2 * b] for b in range(len(stamps) // 2)]
    wait = [stamps[2 * b + 2] - stamps[2 * b + 1] for b in range((len(stamps) - 1) // 2)]
    print(f"step {i:2d} total {stamps[-1] / 1e3:7.1f} us  work " + " ".join(f"{w / 1e3:6.1f}" for w in work)
          + "  | barrier " + " ".join(f"{w / 1e3:5.1f}" for w in wait))
