"""B200-native (sm_100a, FP64) tau-preconditioned GMRES for the CN / quasi-compact
discretisation of the d-dimensional Riesz space fractional diffusion equation
(arXiv 2404.10221).

The product is ``librsfde.so`` (C ABI in ``include/rsfde.h``); ``solver.RsfdeSolver`` is a
thin ctypes binding over it.  ``inputs`` holds the seeded synthetic problem data.
"""
__all__ = ["RsfdeSolver"]


def __getattr__(name):
    if name == "RsfdeSolver":
        from .solver import RsfdeSolver
        return RsfdeSolver
    raise AttributeError(name)
