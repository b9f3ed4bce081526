"""synth -- seeded synthetic inputs shared by the oracle tests, the GPU tests and bench.py.

This module holds none of the method's arithmetic: it only draws plaintext values (coordinates,
intervals, rectangles, identifiers, payload bits) with the shapes and value distributions of
BASELINE.json's five configs.  The paper's four datasets are absent;
these stand in for them and no dataset record is reproduced.
"""
from .workloads import CONFIGS, Workload, make_workload, nand_inputs  # noqa: F401
