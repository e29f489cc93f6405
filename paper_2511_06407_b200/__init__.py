"""B200-native SoftAbs RMHMC inner loop for hierarchical reduced-rank GP models.

Drop-in for the reference package ``softabs_gp`` (arxiv 2511.06407) on its hot
path: the posterior evaluator, the SoftAbs metric with warm-started Jacobi
eigendecompositions, the generalized leapfrog and the MH chain run on the GPU
through libsgp.so (hand-written sm_100a CUDA behind a C ABI, include/sgp.h).
Host-side pieces (model specs, simulators, RNG, statistics) mirror the
reference's API.  Importing the package does not touch the GPU; the first
device call loads libsgp.so and fails loudly if it or the GPU is missing.
"""

from .rrgp import (  # noqa: F401
    Dataset, KernelSpec, ModelSpec, SchemaError, TruthRecord, build_model, feature_value,
    read_csv, simulate_logistic, simulate_meanvar, spectral_variance, write_csv,
)
from .metric import (  # noqa: F401
    BetancourtCache, JacobiError, MetricState, build_cache, dynamic_eigendecompose, metric_apply,
    metric_apply_inverse, metric_from_hessian, sample_momentum, softabs, softabs_deriv,
    static_eigendecompose, t_matrix, w1_matrix, w2_matrix,
)
from .posterior import (  # noqa: F401
    DivergenceError, DomainError, ParamVector, PosteriorTarget, QuadraticTarget, dense_oracle, gradient,
    hessian, neg_log_posterior, potential_derivatives, trace_contractions,
)
from .sampler import (  # noqa: F401
    ChainConfig, ChainError, ChainRecord, ChainResult, euclidean_hmc_run, grad_q_hamiltonian,
    hamiltonian, leapfrog_step, rank_sum_test, read_jsonl, rmhmc_run, run_chain, run_chains,
    wilcoxon_split_half, write_jsonl,
)
from .evidence import (  # noqa: F401
    EvidenceEstimate, GridSpec, TemperLadder, default_ladder, laplace_full, laplace_grid_oracle,
    thermo_integrate, ti_variance,
)

# the reference's public names (softabs_gp/__init__.py:75-132), plus this package's extras
__all__ = [
    "BetancourtCache", "ChainConfig", "ChainError", "ChainRecord", "ChainResult", "Dataset",
    "DivergenceError", "DomainError", "EvidenceEstimate", "GridSpec", "JacobiError", "KernelSpec",
    "MetricState", "ModelSpec", "ParamVector", "PosteriorTarget", "SchemaError", "TemperLadder",
    "TruthRecord", "build_cache", "build_model", "default_ladder", "dense_oracle",
    "dynamic_eigendecompose", "euclidean_hmc_run", "feature_value", "grad_q_hamiltonian", "gradient",
    "hamiltonian", "hessian", "laplace_full", "laplace_grid_oracle", "leapfrog_step", "metric_apply",
    "metric_apply_inverse", "metric_from_hessian", "neg_log_posterior", "potential_derivatives",
    "rank_sum_test", "read_csv", "read_jsonl", "rmhmc_run", "run_chain", "sample_momentum",
    "simulate_logistic", "simulate_meanvar", "softabs", "softabs_deriv", "spectral_variance",
    "static_eigendecompose", "t_matrix", "thermo_integrate", "ti_variance", "trace_contractions",
    "write_csv", "write_jsonl",
    # extras
    "QuadraticTarget", "run_chains",
]

__version__ = "0.1.0"
