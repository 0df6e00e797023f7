"""CPU oracle (TEST INFRASTRUCTURE ONLY).

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / --impl reference legs may
import anything under oracle/.  The product package never imports it.  See fq_oracle.py.
"""
from .fq_oracle import *  # noqa: F401,F403
from . import fq_oracle  # noqa: F401
