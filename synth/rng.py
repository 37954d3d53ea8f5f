"""Counter-based generator for the synthetic special-quadrature blocks.

The near-correction blocks B of the paper (Eq. e:nystrom-correction) come
from quadrature tables this build does not construct (SURVEY §2, A9-A12 OUT).  They
are synthesised instead, bit-reproducibly, from SplitMix64 (Steele, Lea & Flood 2014;
Vigna's reference splitmix64.c) evaluated at a counter:

    z_i      = splitmix64 output number i (0-based) of the generator seeded with `seed`
             = mix(seed + (i+1) * 0x9E3779B97F4A7C15)
    u_i      = (z_i >> 11) * 2^-53                        in [0, 1)
    B[p][e]  = ((2 u_i - 1) * sqrt(3)) * s_blk,  i = p * block_len + e

so every entry has zero mean and variance s_blk^2.  The oracle (C) and the CUDA library
each implement this definition on their own; this module is the readable statement of
it, used only by tests (it holds none of the operator's arithmetic).
"""
import numpy as np

_M64 = (1 << 64) - 1
GOLDEN = 0x9E3779B97F4A7C15
SQRT3 = 1.7320508075688772  # correctly rounded sqrt(3)


def _mix(z):
    z = ((z ^ (z >> 30)) * 0xBF58476D1CE4E5B9) & _M64
    z = ((z ^ (z >> 27)) * 0x94D049BB133111EB) & _M64
    return z ^ (z >> 31)


def splitmix64(seed: int, i: int) -> int:
    """Output number i (0-based) of SplitMix64 started from state `seed`."""
    return _mix((seed + (i + 1) * GOLDEN) & _M64)


def splitmix64_u01(seed: int, i: int) -> float:
    return (splitmix64(seed, i) >> 11) * (1.0 / 9007199254740992.0)


def block_entry_reference(seed: int, flat_index: int, s_blk: float) -> float:
    u = splitmix64_u01(seed, flat_index)
    return ((2.0 * u - 1.0) * SQRT3) * s_blk


def splitmix64_array(seed: int, idx: np.ndarray) -> np.ndarray:
    """Vectorised SplitMix64 (uint64 wrap-around arithmetic)."""
    with np.errstate(over="ignore"):
        z = np.uint64(seed) + (idx.astype(np.uint64) + np.uint64(1)) * np.uint64(GOLDEN)
        z = (z ^ (z >> np.uint64(30))) * np.uint64(0xBF58476D1CE4E5B9)
        z = (z ^ (z >> np.uint64(27))) * np.uint64(0x94D049BB133111EB)
        return z ^ (z >> np.uint64(31))


def block_entries_array(seed: int, idx: np.ndarray, s_blk: float) -> np.ndarray:
    u = (splitmix64_array(seed, idx) >> np.uint64(11)).astype(np.float64) * (1.0 / 9007199254740992.0)
    return ((2.0 * u - 1.0) * SQRT3) * s_blk
