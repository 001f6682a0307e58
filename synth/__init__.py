"""Seeded synthetic input generators shared by tests, bench.py and the oracle driver.

This package holds NO arithmetic of the LLEP method (no planner, no dispatch, no
FFN).  It only produces inputs: routing ids, gate weights, tokens and expert
weights, with the structure of the paper's workloads (§5.1).
Both the CUDA path (via torch, on the device) and the oracle (via numpy, on the
host) draw the same values from the counter-based generator in `workload.py`.
"""
from .workload import *  # noqa: F401,F403
