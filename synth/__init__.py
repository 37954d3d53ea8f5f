"""Seeded synthetic input generator shared by the CUDA path, the oracle and the bench.

This package holds NO arithmetic of the method on the hot path (no upsampling,
no kernel sums, no corrections, no projector).  It only produces the problem
statement the paper's operator takes as input (§3.1 "Surface
discretization", and Eq. e:nystrom-no-correction's weights,
P:L870-876): node coordinates, outward normals, quadrature weights, densities,
near-lists, CFIE mixing parameters, and the counter-based generator that both
sides use to synthesise the special-quadrature blocks.

Every input is seeded; recipes are stated in DESIGN.md ("Input recipe").
"""
from .rng import splitmix64, splitmix64_u01, block_entry_reference
from .geometry import (Body, torus_body, trefoil_body, discretize, gauss_legendre_np,
                       random_rotation)
from .configs import CONFIGS, make_config, make_torus_problem, Problem, pin_torus
from .nearlist import build_near_csr

__all__ = ["splitmix64", "splitmix64_u01", "block_entry_reference", "Body", "torus_body",
           "trefoil_body", "discretize", "gauss_legendre_np", "random_rotation", "CONFIGS",
           "make_config", "make_torus_problem", "Problem", "pin_torus", "build_near_csr"]
