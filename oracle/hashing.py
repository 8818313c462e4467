"""O1 - counter-based hash used for every random choice of the method.

The paper only says nodes and edges are "randomly sampled" (§2.1;
Alg. 1 lines 391 and 396).  Reading R9/R10 in DESIGN.md fixes the generator:
the splitmix64 output function (Steele, Lea, Flood 2014; public-domain reference
by S. Vigna) applied to counters, so that GPU and oracle draw identical
"random" keys without sharing code.

All arithmetic is modulo 2**64 (numpy uint64 wraps).  Written out with Python
ints as well, so a reader can check it by eye.
"""
import numpy as np

MASK64 = (1 << 64) - 1
GAMMA = 0x9E3779B97F4A7C15
M1 = 0xBF58476D1CE4E5B9
M2 = 0x94D049BB133111EB


def mix64_int(z: int) -> int:
    """splitmix64 finaliser on one Python int."""
    z &= MASK64
    z = ((z ^ (z >> 30)) * M1) & MASK64
    z = ((z ^ (z >> 27)) * M2) & MASK64
    return z ^ (z >> 31)


def smx_int(x: int) -> int:
    """smx(x) = mix64(x + gamma): the splitmix64 output for state x."""
    return mix64_int((x + GAMMA) & MASK64)


def key_node_int(seed: int, g: int) -> int:
    """key_node(seed, g) = smx(smx(seed) ^ g)  (R9)."""
    return smx_int(smx_int(seed) ^ g)


def key_edge_int(seed: int, gi: int, gj: int) -> int:
    """key_edge(seed, gi, gj) = smx(smx(smx(seed) ^ gi) ^ gj)  (R10)."""
    return smx_int(smx_int(smx_int(seed) ^ gi) ^ gj)


# ---- vectorised numpy versions (same formulas, uint64 wrap-around) ----------

def _mix64(z: np.ndarray) -> np.ndarray:
    z = np.asarray(z, dtype=np.uint64)
    with np.errstate(over="ignore"):
        z = (z ^ (z >> np.uint64(30))) * np.uint64(M1)
        z = (z ^ (z >> np.uint64(27))) * np.uint64(M2)
    return z ^ (z >> np.uint64(31))


def smx(x: np.ndarray) -> np.ndarray:
    x = np.asarray(x, dtype=np.uint64)
    with np.errstate(over="ignore"):
        return _mix64(x + np.uint64(GAMMA))


def key_node(seed: int, g: np.ndarray) -> np.ndarray:
    s = np.uint64(smx_int(seed))
    return smx(s ^ np.asarray(g).astype(np.uint64))


def key_edge(seed: int, gi, gj) -> np.ndarray:
    s = np.uint64(smx_int(seed))
    a = smx(s ^ np.asarray(gi).astype(np.uint64))
    return smx(a ^ np.asarray(gj).astype(np.uint64))
