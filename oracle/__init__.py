"""CPU oracle for the LE-MPR hot path — TEST INFRASTRUCTURE ONLY.

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / --impl reference
legs may import this package. The product package (paper_2212_01317_b200) never
imports it and shares no code with it. See oracle/mpr_oracle.c for the citations
and docs/ARITH.md for the arithmetic both sides follow independently.
"""
from .oracle import *  # noqa: F401,F403
