"""The C-ABI library loads and exports every symbol include/slq_b200.h declares (no GPU needed)."""
import ctypes
import os
import re

import pytest

from oracle import pcg64
from paper_2003_01282_b200 import _lib

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def declared_symbols():
    text = open(os.path.join(ROOT, "include", "slq_b200.h")).read()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"\b(slq_[a-z0-9_]+)\s*\(", text)))


def test_library_exports_every_declared_symbol():
    lib = _lib.load()
    names = declared_symbols()
    assert len(names) >= 20
    for name in names:
        assert hasattr(lib, name), name
    assert set(names) == set(_lib.exported_symbols())


def test_build_info_names_sm100a():
    assert b"sm_100a" in _lib.load().slq_build_info()


@pytest.mark.parametrize("seed,index", [(0, 0), (0, 1), (7, 5), (123, 99), (2**40 + 3, 17), (5, 2**33 + 1)])
def test_host_probe_state_matches_seedsequence(seed, index):
    out = (ctypes.c_uint64 * 4)()
    assert _lib.load().slq_probe_state(seed, index, out) == 0
    state, inc = pcg64.pcg64_initial_state(seed, index)
    assert (out[0] << 64) | out[1] == state
    assert (out[2] << 64) | out[3] == inc


def test_sm100a_cubin_embedded():
    import subprocess

    r = subprocess.run(["cuobjdump", "--list-elf", _lib.LIB_PATH], capture_output=True, text=True)
    if r.returncode != 0:
        pytest.skip("cuobjdump unavailable")
    assert "sm_100a" in r.stdout


@pytest.mark.parametrize("seed,sample,level", [(0, 0, 0), (0, 12345, 7), (2**63 + 5, 2**40, 26), (17, 3, 63)])
def test_host_rmat_uniform_matches_numpy_restatement(seed, sample, level):
    import numpy as np

    from paper_2003_01282_b200.synth import _splitmix64

    out = ctypes.c_double()
    assert _lib.load().slq_rmat_uniform_host(seed, sample, level, ctypes.byref(out)) == 0
    with np.errstate(over="ignore"):
        base = _splitmix64(np.array([np.uint64(seed) ^ np.uint64(0xD1B54A32D192ED03)], dtype=np.uint64))
        h = _splitmix64(base ^ (np.uint64(sample) * np.uint64(64) + np.uint64(level)))[0]
    assert out.value == float(h >> np.uint64(11)) / 2.0**53


@pytest.mark.parametrize("seed,index", [(0, 3), (2**64 - 1, 0), (2**64, 5), (2**70 + 12345, 2**33 + 1),
                                        (2**127 + 9, 1), (2**128 + 1, 2), (2**255 + 77, 4)])
def test_seeded_probe_state_matches_numpy_for_any_seed(seed, index):
    """slq_seed carries the seed's uint32 entropy words exactly as numpy's SeedSequence splits the
    Python int (slq.py:70 accepts any non-negative int): the PCG64 state equals numpy's."""
    import numpy as np

    out = (ctypes.c_uint64 * 4)()
    assert _lib.load().slq_probe_state_seeded(_lib.seed_arg(seed), index, out) == 0
    st = np.random.PCG64(np.random.SeedSequence(entropy=seed, spawn_key=(index,))).state["state"]
    assert (out[0] << 64) | out[1] == st["state"]
    assert (out[2] << 64) | out[3] == st["inc"]
    if seed < 2**64:
        ref = (ctypes.c_uint64 * 4)()
        assert _lib.load().slq_probe_state(seed, index, ref) == 0
        assert list(ref) == list(out)


def test_seed_arg_rejects_negative_and_oversized():
    with pytest.raises(ValueError):
        _lib.seed_arg(-1)
    with pytest.raises(ValueError):
        _lib.seed_arg(2**256)
