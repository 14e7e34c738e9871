"""B200-native batched alternating-minimisation trajectory optimiser (arXiv 2109.13030).

The product path is libbmc.so (C-ABI in include/bmc.h, fused sm_100a kernel in
csrc/); this package holds its thin ctypes binding (bmc.py), the sharded
multi-GPU wrapper (distributed.py) and the receding-horizon MPC loop around
the solver (mpc.py).  Nothing here imports the test oracle.
"""
from .bmc import BmcError, Solver, load_library, solver_for  # noqa: F401

__all__ = ["Solver", "BmcError", "load_library", "solver_for"]
