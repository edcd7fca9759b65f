"""Parameter packing for the C ABI (include/sr_block.h "Network"): theta = [W_0 (row-major), b_0, W_1, b_1, ...]."""
from __future__ import annotations

import numpy as np


def pack(params) -> np.ndarray:
    return np.concatenate([np.concatenate([np.asarray(w).ravel(), np.asarray(b)]) for w, b in params]).astype(
        np.complex128)


def widths_of(params):
    return [params[0][0].shape[1]] + [w.shape[0] for w, _ in params]
