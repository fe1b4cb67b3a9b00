"""ORACLE / TEST INFRASTRUCTURE ONLY — never imported by the product package.

Pure-integer restatement of the probe stream the reference draws at
``slq.py:63-72`` (``/root/reference/pkg/src/spectrace/slq.py``):

    seq = np.random.SeedSequence(entropy=cfg.seed, spawn_key=(index,))
    rng = np.random.default_rng(seq)
    v   = rng.integers(0, 2, size=n).astype(np.float64) * 2.0 - 1.0

The arithmetic lives in numpy (un-vendored third-party dependency; unpinned
``numpy>=1.24`` at ``pkg/pyproject.toml:11``; 2.3.5 in this image).  Its
published algorithms are restated here from their definitions:

* SeedSequence (numpy ``bit_generator.pyx``): 4-word uint32 entropy pool built
  with the ``hashmix``/``mix`` functions, then ``generate_state`` expands the
  pool with a second hash stream.
* PCG64 (O'Neill's PCG-XSL-RR 128/64): 128-bit LCG, step then output
  ``rotr64(hi ^ lo, state >> 122)``; seeding via ``pcg_setseq_128_srandom``.
* ``Generator.integers(0, 2)`` (int64): Lemire bounded draw on buffered 32-bit
  halves of the 64-bit stream (low half first); for a range of 2 the result is
  bit 31 of each 32-bit half and nothing is ever rejected.

This module pins the device generator: tests compare it against numpy itself
(the reference's dependency) and against the CUDA kernels.
"""
from __future__ import annotations

MASK32 = 0xFFFFFFFF
MASK64 = (1 << 64) - 1
MASK128 = (1 << 128) - 1

PCG_MULT = 0x2360ED051FC65DA44385DF649FCCF645

_INIT_A = 0x43B0D7E5
_MULT_A = 0x931E8875
_INIT_B = 0x8B51F9DD
_MULT_B = 0x58F38DED
_MIX_L = 0xCA01F9DD
_MIX_R = 0x4973F715
_XSHIFT = 16
_POOL = 4


def _words32(value: int) -> list[int]:
    """Little-endian uint32 words of a non-negative int (0 -> [0])."""
    if value < 0:
        raise ValueError("entropy must be non-negative")
    out = []
    while True:
        out.append(value & MASK32)
        value >>= 32
        if value == 0:
            return out


class _Hasher:
    def __init__(self, const: int):
        self.const = const

    def __call__(self, value: int) -> int:
        value = (value ^ self.const) & MASK32
        self.const = (self.const * _MULT_A) & MASK32
        value = (value * self.const) & MASK32
        return value ^ (value >> _XSHIFT)


def _mix(x: int, y: int) -> int:
    r = (_MIX_L * x - _MIX_R * y) & MASK32
    return r ^ (r >> _XSHIFT)


def seed_sequence_pool(entropy: int, spawn_key: tuple[int, ...]) -> list[int]:
    run = _words32(entropy)
    spawn: list[int] = []
    for k in spawn_key:
        spawn.extend(_words32(k))
    if spawn and len(run) < _POOL:
        run = run + [0] * (_POOL - len(run))
    data = run + spawn
    h = _Hasher(_INIT_A)
    pool = [h(data[i]) if i < len(data) else h(0) for i in range(_POOL)]
    for src in range(_POOL):
        for dst in range(_POOL):
            if src != dst:
                pool[dst] = _mix(pool[dst], h(pool[src]))
    for src in range(_POOL, len(data)):
        for dst in range(_POOL):
            pool[dst] = _mix(pool[dst], h(data[src]))
    return pool


def seed_sequence_words64(pool: list[int], n_words: int) -> list[int]:
    const = _INIT_B
    out32 = []
    for i in range(2 * n_words):
        v = (pool[i % _POOL] ^ const) & MASK32
        const = (const * _MULT_B) & MASK32
        v = (v * const) & MASK32
        out32.append(v ^ (v >> _XSHIFT))
    return [out32[2 * k] | (out32[2 * k + 1] << 32) for k in range(n_words)]


def pcg64_initial_state(seed: int, index: int) -> tuple[int, int]:
    """(state, inc) of PCG64(SeedSequence(entropy=seed, spawn_key=(index,)))."""
    w = seed_sequence_words64(seed_sequence_pool(seed, (index,)), 4)
    initstate = (w[0] << 64) | w[1]
    initseq = (w[2] << 64) | w[3]
    inc = ((initseq << 1) | 1) & MASK128
    state = (0 * PCG_MULT + inc) & MASK128
    state = (state + initstate) & MASK128
    state = (state * PCG_MULT + inc) & MASK128
    return state, inc


def pcg64_outputs(state: int, inc: int, count: int) -> list[int]:
    out = []
    for _ in range(count):
        state = (state * PCG_MULT + inc) & MASK128
        hi, lo = state >> 64, state & MASK64
        rot = state >> 122
        x = hi ^ lo
        out.append(((x >> rot) | (x << ((64 - rot) & 63))) & MASK64)
    return out


def rademacher(seed: int, index: int, n: int) -> list[float]:
    """Probe ``index`` of length n as +-1.0 floats (pure Python; small n only)."""
    state, inc = pcg64_initial_state(seed, index)
    raw = pcg64_outputs(state, inc, (n + 1) // 2)
    vals = []
    for k in range(n):
        word = raw[k >> 1]
        half = (word & MASK32) if (k & 1) == 0 else (word >> 32)
        vals.append(1.0 if (half >> 31) & 1 else -1.0)
    return vals
