"""B200-native MGRIT/Parareal hot path for 1D periodic linear advection (arXiv:1910.03726).

Compute runs in libmgrit.so (hand-written sm_100a CUDA behind the C ABI in
include/mgrit.h); this package is the thin Python binding plus host-side set-up.
"""
from . import binding  # noqa: F401
from .binding import MGRIT, MgritError, fill_guess, scheme_coefficients  # noqa: F401
