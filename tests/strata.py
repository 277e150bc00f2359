"""Row / coefficient samples for the full-size parity tests that cover the
GEMMs' structure: both CTAs of a 256-row pair tile
(row % 256 < 128 and >= 128), all four TMEM lane quarters of a CTA
((row % 128) // 32), the first, last and interior row blocks, and rows next to
64-row K-block and 256-row tile boundaries.  Pure index bookkeeping; no
arithmetic of the method."""
from __future__ import annotations

import numpy as np


def stratified_rows(N: int, min_rows: int = 64) -> np.ndarray:
    nb = (N + 255) // 256
    blocks = sorted({0, 1, nb // 3, nb // 2, (2 * nb) // 3, max(nb - 2, 0), nb - 1})
    rows = set()
    for a in blocks:
        for h in (0, 1):          # CTA of the pair
            for q in range(4):    # TMEM lane quarter
                lane = (7 * a + 13 * h + 5 * q) % 32
                i = 256 * a + 128 * h + 32 * q + lane
                if i < N:
                    rows.add(i)
    # tile / K-block boundaries and the ragged end
    for i in (63, 64, 127, 128, 255, 256, N - 129, N - 128, N - 65, N - 64, N - 2, N - 1):
        if 0 <= i < N:
            rows.add(i)
    rng = np.random.default_rng(N)
    while len(rows) < min(min_rows, N):
        rows.add(int(rng.integers(0, N)))
    return np.array(sorted(rows), dtype=np.int64)


def strata_covered(rows: np.ndarray, N: int) -> dict:
    """Which (CTA, lane quarter) cells and which row blocks a sample touches."""
    cells = {(int(i % 256) // 128, int(i % 128) // 32) for i in rows}
    blocks = {int(i) // 256 for i in rows}
    return {"cells": cells, "first": 0 in blocks, "last": (N - 1) // 256 in blocks}
