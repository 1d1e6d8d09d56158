"""CPU oracle package — TEST INFRASTRUCTURE ONLY (see spectrain_oracle.py header).

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / --impl
reference leg may import it. The product package never does.
"""
from .spectrain_oracle import *  # noqa: F401,F403
