"""B200-native IGA-FEM integration + assembly (hot path of arXiv 2207.00280).

Drop-in for the reference package ``igabench`` on its integration and assembly
path: same public names and signatures (igabench/__init__.py:10-58), with the
numerics executed by hand-written sm_100a CUDA kernels in
``lib/libiga_b200.so`` (C-ABI: ``include/iga_b200.h``).  There is no CPU
fallback.
"""

__version__ = "0.1.0"

from .assembly import (
    GlobalGram,
    assemble,
    dof_index,
    element_dofs,
    sparsity_row_bound,
    spmv,
    symbolic_pattern,
    write_matrix_market,
)
from .integrators import (
    ElementMatrix,
    SumFactBuffers,
    canonical_pairs,
    default_rule,
    element_tables,
    flop_count,
    integrate_element_classical,
    integrate_element_sumfact,
)
from .operator import MatrixFreeOperator, cg
from .mesh import QuadratureRule, element_list, gauss_rule, knot_rule, local_index, support_set
from .runtime import (
    ExecutionTrace,
    IntegrationRuntime,
    RunConfig,
    RunResult,
    grams_bitwise_equal,
    run_integration,
    run_within_element,
)
from .splines import (
    BasisValues,
    KnotVector,
    basis_derivative_table,
    basis_value_table,
    eval_basis,
    eval_basis_many,
    eval_basis_order0,
    eval_nonzero_basis,
    eval_nonzero_basis_derivatives,
    check_knots,
    find_element,
    make_general_knot_vector,
    make_knot_vector,
)

__all__ = [
    "BasisValues",
    "ElementMatrix",
    "ExecutionTrace",
    "GlobalGram",
    "IntegrationRuntime",
    "KnotVector",
    "MatrixFreeOperator",
    "QuadratureRule",
    "RunConfig",
    "RunResult",
    "SumFactBuffers",
    "assemble",
    "basis_derivative_table",
    "basis_value_table",
    "canonical_pairs",
    "cg",
    "default_rule",
    "dof_index",
    "element_dofs",
    "element_list",
    "element_tables",
    "eval_basis",
    "eval_basis_many",
    "eval_basis_order0",
    "eval_nonzero_basis",
    "eval_nonzero_basis_derivatives",
    "find_element",
    "flop_count",
    "gauss_rule",
    "knot_rule",
    "make_general_knot_vector",
    "check_knots",
    "grams_bitwise_equal",
    "integrate_element_classical",
    "integrate_element_sumfact",
    "local_index",
    "make_knot_vector",
    "run_integration",
    "run_within_element",
    "sparsity_row_bound",
    "spmv",
    "support_set",
    "symbolic_pattern",
    "write_matrix_market",
]
