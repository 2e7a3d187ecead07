"""The comparator lives with the oracle (oracle/parity.py) so bench.py can use it too."""

from oracle.parity import *  # noqa: F401,F403
from oracle.parity import NEAR_TIE, NOISE_RESIDUAL, RTOL, ATOL_REL_X, ParityReport, compare  # noqa: F401
