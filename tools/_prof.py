import sys, json; sys.path.insert(0, '.')
import torch
from paper_2003_01282_b200 import _lib, synth
from paper_2003_01282_b200.device import DeviceGraph
dev = torch.device("cuda", 0)
dg = DeviceGraph(synth.sbm(100_000, 10, 1e-3, 1e-5, seed=0), dev)
for dt in ("f64", "f32"):
    for _ in range(2):
        dg.rules("normalized_laplacian", 0, 0, 100, 15, dtype=dt).check()
    _lib.profile_begin()
    dg.rules("normalized_laplacian", 0, 0, 100, 15, dtype=dt)
    torch.cuda.synchronize()
    print(dt, json.dumps({k: round(v["ms"], 3) for k, v in _lib.profile_end().items() if v["launches"]}))
