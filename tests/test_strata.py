"""The stratified row sample of the full-size GPU parity tests (CPU check)."""
import seeded_inputs as si
from strata import strata_covered, stratified_rows


def test_stratified_rows_cover_the_tiles():
    """The sample used below covers both CTAs x 4 lane quarters and the first
    and last row blocks at configs 3 and 4 (and has >= 64 rows)."""
    for name in ("c3_n12_2d12", si.BENCH_CONFIG):
        N = si.CONFIGS[name].N
        rows = stratified_rows(N)
        cov = strata_covered(rows, N)
        assert rows.size >= 64 and cov["first"] and cov["last"]
        assert cov["cells"] == {(h, q) for h in (0, 1) for q in range(4)}
