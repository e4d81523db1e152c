"""B200-native shift-invert Krylov eigensolver for quadratic pencils from IGA/rIGA
discretisations (arXiv 2112.14064). Host C++ + sm_100a CUDA behind the C-ABI in
include/rq_b200.h; this package is the Python mirror of the reference's
sparsela/eig operations."""
from ._lib import LIB_PATH, RqError  # noqa: F401
from .eig import (EigenPair, GeneralizedHermitianSolver, ShiftInvertOperator, apply_operator,  # noqa: F401
                  arnoldi_run, b_inner, build_operator, krylov_schur_restart, ritz_extract, scale_pencil,
                  solve_generalized_hermitian, solve_quadratic, solve_quadratic_complex)
from .pencil import CURL, DIV, QuadraticPencil, assemble, assemble_acoustic, assemble_em, baseline_config  # noqa: F401
from .io import (eigenpairs_json, load_eigenpairs, read_matrix_market,  # noqa: F401
                 write_eigenpairs, write_matrix_market, write_matrix_market_vector, write_pencil)
from .sparsela import (Factorization, Ordering, lu_factorize,  # noqa: F401
                       nested_dissection_order, solve_factored)
