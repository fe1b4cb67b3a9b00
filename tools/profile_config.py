"""Per-kernel-class device time (and launches) of one signature's rules on a BASELINE config:
    python tools/profile_config.py c1|c2|c4 [--dtype f64]"""
import argparse
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

from paper_2003_01282_b200 import _lib
from paper_2003_01282_b200.device import DeviceGraph
from run_config import CONFIGS, KIND   # noqa: E402  (tools/ on sys.path when run as a script)

ap = argparse.ArgumentParser()
ap.add_argument("config")
ap.add_argument("--dtype", default="f64")
args = ap.parse_args()
cfg = CONFIGS[args.config]
dev = torch.device("cuda", 0)
dg = DeviceGraph(cfg["make"](), dev)
out = {"config": args.config, "dtype": args.dtype}
for kind in cfg["kinds"]:
    for _ in range(3):
        dg.rules(KIND[kind], 0, 0, cfg["n_v"], cfg["s"], dtype=args.dtype).check()
    torch.cuda.synchronize()
    _lib.profile_begin()
    dg.rules(KIND[kind], 0, 0, cfg["n_v"], cfg["s"], dtype=args.dtype)
    torch.cuda.synchronize()
    out[kind] = {k: {"ms": round(v["ms"], 4), "launches": v["launches"]} for k, v in _lib.profile_end().items()
                 if v["launches"]}
print(json.dumps(out))
