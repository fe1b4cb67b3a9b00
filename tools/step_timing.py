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
which = sys.argv[1] if len(sys.argv) > 1 else "c2"
if which == "c1":
    dg, NV, S = DeviceGraph(synth.barabasi_albert(1000, 3, seed=0), dev), 10, 10
else:
    dg, NV, S = DeviceGraph(synth.sbm(100_000, 10, 1e-3, 1e-5, seed=0), dev), 100, 15
for _ in range(3):
    dg.rules("normalized_laplacian", 0, 0, NV, S).check()
torch.cuda.synchronize()
lib = _lib.load()
STRIDE = 32 + 4 * 160
buf = (ctypes.c_ulonglong * (STRIDE * 128))()
lib.slq_debug_step_times.restype = ctypes.c_int
n = lib.slq_debug_step_times(buf, STRIDE * 128)
full = np.array(buf[:n], dtype=np.float64).reshape(128, STRIDE)
t = full[:, :32]
for i in range(S - 1):
    row = t[i]
    k = [j for j in range(32) if row[j] > 0]
    stamps = row[:max(k) + 1] - row[0]
    work = [stamps[2 * b + 1] - stamps[2 * b] for b in range(len(stamps) // 2)]
    wait = [stamps[2 * b + 2] - stamps[2 * b + 1] for b in range((len(stamps) - 1) // 2)]
    print(f"step {i:2d} total {stamps[-1] / 1e3:7.1f} us  work " + " ".join(f"{w / 1e3:6.1f}" for w in work)
          + "  | barrier " + " ".join(f"{w / 1e3:5.1f}" for w in wait))

# per-CTA end of the two streaming phases (relative to CTA 0's kernel start), for the last steps
for i in (0, (S - 1) // 2, S - 2):
    cta = full[i, 32:32 + 4 * 148].reshape(148, 4)
    cta = cta[cta[:, 0] > 0] if (cta[:, 0] > 0).any() else cta
    a_end = (cta[:, 1] - full[i, 0]) / 1e3
    c_end = (cta[:, 2] - full[i, 0]) / 1e3
    start = (cta[:, 0] - full[i, 0]) / 1e3
    slow_a = np.argsort(a_end)[-8:]
    print(f"step {i}: start spread {start.max() - start.min():.1f} us; phase A end min/med/max "
          f"{a_end.min():.1f}/{np.median(a_end):.1f}/{a_end.max():.1f}; slowest CTAs {sorted(slow_a.tolist())}; "
          f"phase C end min/med/max {c_end.min():.1f}/{np.median(c_end):.1f}/{c_end.max():.1f}; "
          f"slowest {sorted(np.argsort(c_end)[-8:].tolist())}")
