"""paper_1108_1688_b200 — B200-native Douglas-ADI solver for the 3D HJM-SV
pricing PDE of arXiv 1108.1688, a drop-in for the reference's run()/douglas_step
path behind a C-ABI (include/hjmsv_b200.h).

The compute path is the in-tree CUDA library lib/libhjmsv_b200.so (sm_100a);
importing the solver API without it raises ImportError — there is no CPU path.
"""
from . import _abi  # noqa: F401
from .problem import AxisSpec, ProblemSpec, SolverConfig, mix_seed  # noqa: F401
from .api import (Solver, run, price, mc_price, apply_operator, douglas_step, thomas_batch,  # noqa: F401
                  batch_run, device_count, HjmsvError, InvalidArgument, DomainError, LogicError,
                  SolverRuntimeError, SingularPivot, NonFinite, Diverged, Unsupported, CudaError)
from . import workloads  # noqa: F401
from . import drivers  # noqa: F401

__all__ = ["AxisSpec", "ProblemSpec", "SolverConfig", "Solver", "run", "price", "apply_operator",
           "douglas_step", "thomas_batch", "batch_run", "device_count", "workloads"]
