import hashlib

import numpy as np


def sha(a) -> str:
    """SHA-256 of the canonical little-endian float64 bytes (tests/golden/make_golden.py)."""
    return hashlib.sha256(np.ascontiguousarray(a, dtype="<f8").tobytes()).hexdigest()
