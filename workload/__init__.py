"""Seeded synthetic inputs (Jacobians, right-hand sides, random vectors) shared
by the oracle tests, the GPU tests and bench.py.  Contains no BF-AMG-GMRES
arithmetic (see workload/twophase.py docstring)."""
from .twophase import (Problem, CapillaryModel, BSR2, residual, jacobian, harmonic_face_perm,
                       jacobian_slots, DAY, G_ACC, EPS_S)
from .configs import make_problem, make_system, CONFIG_NAMES
from .vectors import seeded_vector
from .newton import newton_sequence

__all__ = ["Problem", "CapillaryModel", "BSR2", "residual", "jacobian", "harmonic_face_perm",
           "jacobian_slots", "make_problem", "make_system", "seeded_vector", "newton_sequence", "CONFIG_NAMES",
           "DAY", "G_ACC", "EPS_S"]
