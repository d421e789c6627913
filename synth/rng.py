"""Counter-based splitmix64 random numbers (vectorised numpy, uint64 wrap-around).

rand_u64(seed, stream, counter) = mix64(key(seed, stream) + (counter + 1) * GOLDEN)
where key(seed, stream) = mix64(mix64(seed) ^ (stream * STREAM_MUL)) and mix64 is the
splitmix64 output finaliser. Pure function of its three arguments, so any element
can be regenerated alone (window-parallel, rank-parallel generation).
"""
import numpy as np

GOLDEN = np.uint64(0x9E3779B97F4A7C15)
STREAM_MUL = np.uint64(0xD1B54A32D192ED03)
_M1 = np.uint64(0xBF58476D1CE4E5B9)
_M2 = np.uint64(0x94D049BB133111EB)


def mix64(z):
    z = np.asarray(z, dtype=np.uint64)
    with np.errstate(over="ignore"):
        z = (z ^ (z >> np.uint64(30))) * _M1
        z = (z ^ (z >> np.uint64(27))) * _M2
        return z ^ (z >> np.uint64(31))


def _key(seed, stream):
    seed = np.asarray(seed, dtype=np.uint64)
    stream = np.asarray(stream, dtype=np.uint64)
    with np.errstate(over="ignore"):
        return mix64(mix64(seed + GOLDEN) ^ (stream * STREAM_MUL))


def rand_u64(seed, stream, counter):
    counter = np.asarray(counter, dtype=np.uint64)
    with np.errstate(over="ignore"):
        return mix64(_key(seed, stream) + (counter + np.uint64(1)) * GOLDEN)


def rand_uniform(seed, stream, counter):
    """Uniform doubles in [0, 1) with 53 random bits."""
    u = rand_u64(seed, stream, counter)
    return (u >> np.uint64(11)).astype(np.float64) * (1.0 / 9007199254740992.0)


def rand_int(seed, stream, counter, lo, hi):
    """Integers uniform on [lo, hi] inclusive (Lemire multiply-shift on 32 high bits)."""
    span = np.asarray(hi, dtype=np.int64) - np.asarray(lo, dtype=np.int64) + 1
    u = (rand_u64(seed, stream, counter) >> np.uint64(32)).astype(np.uint64)
    r = ((u * span.astype(np.uint64)) >> np.uint64(32)).astype(np.int64)
    return np.asarray(lo, dtype=np.int64) + r
