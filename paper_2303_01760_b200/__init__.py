"""hybridnodes-b200: the hybrid scattered-regular RBF-FD hot path of arXiv 2303.01760 on B200.

Drop-in for the hot-path API of the reference package `hybridnodes`
(pkg/src/hybridnodes/__init__.py:3-17): stencils and weights (approx), operator
assembly/application (operators) and the explicit natural-convection step driver
(solver), and node-set generation (generate: lattice fill, advancing front, lattice map;
geometry / config: the domains it fills), all computed by hand-written sm_100a kernels in
libhn.so; `sharded` is the one-process-per-GPU form of the step and of compute_weights
(SURVEY §8(e)).  CLI, config-file parsing and plotting are not part of this package;
`nodesets` provides the seeded Appendix-B inputs for the BASELINE configs.
"""

from .approx import (METHOD_MON, METHOD_NONE, METHOD_RBFFD, MON_SIZE, POLY_COUNT, RBF_SIZE, Laplacian,
                     NormalDerivative, Partial, StencilSpec, WeightRow, WeightTable, boundary_partial_table,
                     classify_methods, compute_weights, condition_number, find_stencil, mon_weights,
                     normal_derivative_table, rbf_fd_weights, select_method)
from .config import CaseConfig, build_domain
from .errors import (ConfigurationError, PoissonConvergenceError, SingularSystemError,
                     SolverDivergenceError)
from .generate import (RegularFill, SpacingFunction, carve_transition, hybrid_discretize, regular_fill,
                       scattered_fill)
from .geometry import (BoundarySet, Circle, DomainSpec, Ellipse, Obstacle, Star, discretize_boundary,
                       signed_distance)
from .nodegen import (KIND_BOUNDARY, KIND_REGULAR, KIND_SCATTERED, ROLE_DIRICHLET, ROLE_INTERIOR,
                      ROLE_NEUMANN, LatticeInfo, Node, NodeSet)
from .operators import FieldState, SparseOperator, apply, assemble, divergence
from .sharded import (HaloPlan, LocalTransport, ShardedStepper, TorchDistTransport, build_halo_plan,
                      compute_weights_sharded, partition_nodes)
from .solver import (DeviceStepper, OperatorSet, PhysicsParams, PoissonSolveSettings, RunResult,
                     TimeControls, apply_temperature_bc, apply_velocity_bc, build_operators,
                     interior_divergence, momentum_predict, nusselt_average, pressure_solve, run,
                     temperature_step, velocity_correct, write_outputs)

__all__ = [name for name in dir() if not name.startswith("_")]
__version__ = "0.1.0"
