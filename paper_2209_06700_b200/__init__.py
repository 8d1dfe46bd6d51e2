"""B200-native hot path of the stage-parallel Radau IIA method (arXiv 2209.06700).

Drop-in for the reference `spirk` package's operator / preconditioner / Krylov / stepper API on
device-resident fp64 tensors; all hot arithmetic runs in libspk (`_spk.so`, sm_100a kernels).
"""

__all__ = ["errors", "tableau", "fem", "multigrid", "krylov", "tensor_ops", "irk", "complex_solver",
           "parallel"]
