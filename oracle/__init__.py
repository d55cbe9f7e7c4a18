"""fp64 CPU oracle (TEST INFRASTRUCTURE ONLY) -- see oracle/tprod_oracle.py for the contract.

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / --impl reference legs may
import this package.  The product path never does.
"""
from .tprod_oracle import *  # noqa: F401,F403
from .tprod_oracle import __all__  # noqa: F401
