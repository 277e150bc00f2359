"""fp64 CPU oracle (TEST INFRASTRUCTURE ONLY -- see oracle.py)."""
from .oracle import OracleIndex, adam_update, basis_count, build, gd_update, host_threads  # noqa: F401
