"""B200-native hot path of the over-parameterised SOS method (arxiv 2410.19844).

Public API (thin binding over the C ABI in include/sos_b200.h):
    SosIndex(n, d)            monomial tables + pair-rank table (device)
    SosPlan(index, r)         forward / backward / loss_grad / step / solve_host
"""
from .binding import SOS_OPT_ADAM, SOS_OPT_GD, SosError, SosIndex, SosPlan, load  # noqa: F401

__all__ = ["SosIndex", "SosPlan", "SosError", "load", "SOS_OPT_GD", "SOS_OPT_ADAM"]
