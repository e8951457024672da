"""CPU oracle (test infrastructure only; see adct_oracle.py header)."""
from .adct_oracle import *  # noqa: F401,F403
