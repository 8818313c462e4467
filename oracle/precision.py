"""Operand precision model of the BF16 mode (reading R18).

The BF16 mode feeds every tensor-core product bf16 operands: the inputs v, e,
the weights, and the kappa_phi activations a1 and h (the operands of the next
product).  The oracle keeps fp64 arithmetic but, in BF16 mode, applies the same
operand rounding to a1 and h, so that the ReLU decisions [a1 > 0], [h > 0]
are taken on the same values on both sides (a floating-point decision must
be taken in the same precision on both sides).  Own implementation of
round-to-nearest-even to bf16 (8 significand bits); pinned against torch's
CPU conversion in tests/test_oracle_layer.py.
"""
import numpy as np


def round_bf16(x) -> np.ndarray:
    """Round to the nearest bf16 value (ties to even); returns float64 values."""
    x32 = np.ascontiguousarray(np.asarray(x, dtype=np.float64).astype(np.float32))
    u = x32.view(np.uint32).astype(np.uint64)
    lsb = (u >> np.uint64(16)) & np.uint64(1)
    r = ((u + np.uint64(0x7FFF) + lsb) >> np.uint64(16)) << np.uint64(16)
    out = (r & np.uint64(0xFFFFFFFF)).astype(np.uint32).view(np.float32)
    out = np.where(np.isfinite(x32), out, x32)
    return out.astype(np.float64)
