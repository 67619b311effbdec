"""Solver configuration/report types (drop-in for diffproj.linsolve's
SolverConfig / SolveReport, linsolve.py:21-42).  The solvers themselves are
device kernels (csrc/dp_kernels.cu: Chronopoulos-Gear PCG and GMRES(m) with
3x3 block-Jacobi preconditioning)."""

from __future__ import annotations

from dataclasses import dataclass, field

from . import _lib

_METHODS = {"auto": 0, "cg": 1, "gmres": 2}


@dataclass
class SolverConfig:
    method: str = "auto"          # auto: CG iff symmetric (adjoint.py:128-133)
    precond: str = "block_jacobi"
    tol: float = 1e-10
    max_iter: int = 2000
    gmres_restart: int = 50

    def __post_init__(self):
        if self.tol <= 0:
            raise ValueError("tol must be positive")
        if self.max_iter < 1:
            raise ValueError("max_iter must be at least 1")

    def to_c(self):
        c = _lib.SolverCfgC()
        c.method = _METHODS.get(self.method, 0)
        c.tol = self.tol
        c.max_iter = self.max_iter
        c.gmres_restart = self.gmres_restart
        return c


@dataclass
class SolveReport:
    residual_history: list = field(default_factory=list)
    converged: bool = False
    diverged: bool = False
    iterations: int = 0
    wall_time: float = 0.0
