"""fp64 CPU oracle for the PROBE MoE hot path — TEST INFRASTRUCTURE ONLY.

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / --impl
reference legs may import this package.  The product path (the CUDA library
and its binding) never imports it, and it imports nothing from the product.
"""
from .probe_oracle import *  # noqa: F401,F403
from .distill_oracle import *  # noqa: F401,F403
