"""Image metrics used for parity reporting (proj/src/image.cpp:101-111)."""
import math

import numpy as np


def psnr(a: np.ndarray, b: np.ndarray) -> float:
    """PSNR over all channels with peak 1, capped at 99 dB (image.cpp:101-111)."""
    if a.shape != b.shape:
        raise ValueError("psnr: shape mismatch")
    d = a.astype(np.float64) - b.astype(np.float64)
    mse = float(np.mean(d * d))
    if mse <= 0:
        return 99.0
    return min(99.0, 10.0 * math.log10(1.0 / mse))
