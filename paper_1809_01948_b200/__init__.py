"""B200-native preconditioned pipelined BiCGStab (arXiv 1809.01948, S. Cools).

Product path: include/pbicgstab.h (C ABI) -> csrc/*.cu (sm_100a kernels + host
driver) -> binding.py (ctypes marshalling).  ``problems`` holds the seeded
synthetic inputs.  Nothing here imports the test oracle (``oracle/``).
"""
from .binding import PbicgError, Solver, SolveResult, lib  # noqa: F401

__all__ = ["Solver", "SolveResult", "PbicgError", "lib"]
