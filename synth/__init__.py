"""Seeded synthetic inputs (quadrature sets, C1..C5, random problems).

The one module both the oracle side and the CUDA side may import: it holds no
sweep, solve or closure arithmetic — only the problem data the paper's problem
statement takes as input.
"""
from .configs import Problem, config, n_bnode, bnode_index, random_problem, replicate_groups  # noqa: F401
from .quadrature import gauss_legendre, product_set, slab_set  # noqa: F401
