"""Oracle (test infrastructure only): plain fp64 CPU implementation of the paper's algorithms.

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / --impl reference legs may
import this package.  The product path (paper_1804_07531_b200) never does.
"""
from .rsvd_oracle import *  # noqa: F401,F403
