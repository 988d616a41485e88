"""Seeded synthetic inputs shaped like the paper's workloads (BASELINE.json configs).

Shared by the oracle tests and by the CUDA path's tests/bench: it produces the
BYTES both sides consume and contains none of the method's arithmetic (no
Gaussian projection, no SVD of a sketch, no Krylov step).  Generation uses
torch (CPU or CUDA) only for speed; the recipe is in DESIGN.md §Inputs.
"""
from .generate import CONFIGS, Problem, make_problem  # noqa: F401
