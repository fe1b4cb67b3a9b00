"""bench.py host logic that needs no GPU: the CPU arms' samplers and the reference arm's JSON line."""
import json
import os
import subprocess
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import bench  # noqa: E402
from oracle import slq_oracle as O  # noqa: E402
from paper_2003_01282_b200 import synth  # noqa: E402


def test_row_sampler_is_the_oracle_operator_on_its_rows():
    """The C5 CPU sample (every 8th row of the normalized-Laplacian apply, full-length vectors) is the
    oracle operator's arithmetic on those rows, bit for bit."""
    g = synth.rmat(14, 16, seed=0)
    off, cols = np.asarray(g.row_offsets), np.asarray(g.col_indices).astype(np.int32)
    apply, alpha, nnz_s = bench.cpu_row_sample_operator(off, cols, g.n, 8)
    x = O.draw_probes(g.n, 0, [0, 1, 2])
    full = O.make_block_operator(g, O.NORMALIZED_LAPLACIAN).apply(x)
    assert np.array_equal(apply(x), full[::8])
    assert nnz_s == int(sum(off[r + 1] - off[r] for r in range(0, g.n, 8)))
    v, dt = bench.cpu_row_sample((apply, alpha, nnz_s, g.n), g.n, 2, 2)
    assert v > 0 and dt > 0


def test_reference_arm_line_matches_our_config():
    """`bench.py --impl reference` prints one JSON line with the contract's keys and the SAME config
    dict as our arm (config_dict), so the driver can pair the two lines."""
    r = subprocess.run([sys.executable, "bench.py", "--impl", "reference", "--config", "c2", "--steps", "1",
                        "--warmup", "3"], cwd=ROOT, capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stderr[-2000:]
    line = json.loads(r.stdout.strip().splitlines()[-1])
    assert line["impl"] == "reference"
    for key in ("metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better", "scaling",
                "dtype", "config", "cpu_baseline", "e2e"):
        assert key in line, key
    assert line["config"] == json.loads(json.dumps(bench.config_dict(bench.CONFIGS["c2"], 1)))
    assert line["e2e"]["h2d_bytes_per_step"] == 0 and line["cpu_baseline"]["kind"] == "port"
