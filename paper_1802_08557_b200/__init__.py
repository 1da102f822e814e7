"""B200-native batched two-phase dense simplex (Gurung & Ray, arXiv 1802.08557).

Drop-in for the batched-solve path of the reference package ``batchlp``
(/root/reference/pkg/src/batchlp/__init__.py:3-12,37): the same names,
signatures, exceptions and result layout for ``batch_solve`` / ``solve`` and
their types, with the simplex itself running as hand-written sm_100a CUDA in
libblp.so (C ABI: include/blp.h).  There is no CPU fallback.

Packed fast paths: ``batch_solve_arrays`` (A [B,m,n], b [B,m], c [B,n]) and
``support_batch`` (one polytope, many objective directions).  The paper's
second kernel, batched hyper-rectangle LPs (Eq. 7), is ``solve_box_batch`` /
``box_batch_arrays`` (reference boxlp.py).  General-form ingest (GeneralLP,
MPS files) lowers to packed batches and maps results back (general.py, mps.py).
"""
from .batch import (
    REFERENCE_GPU_BLOCK_COLS,
    BatchArrays,
    BatchConfig,
    BatchReport,
    BatchTooLarge,
    ChunkPlan,
    HeterogeneousBatch,
    batch_solve,
    batch_solve_arrays,
    lp_memory_bytes,
    plan_chunks,
    support_batch,
)
from .boxlp import BoxArrays, BoxLP, BoxSolution, InvalidBox, box_batch_arrays, solve_box, solve_box_batch
from .certify import ORACLE_TOL, Certificate, CertificateBatch, certify_batch, check_certificate
from .general import (GeneralBatch, GeneralLP, InfeasibleBounds, Relation, Sense, VariableMap,
                      batch_solve_general, recover_batch, solve_general, standardize, standardize_batch)
from .model import SolveOutcome, StandardFormLP, Status, standard_form, validate
from .mps import MpsModel, ParseError, UnsupportedFeature, lower_to_general, parse_mps
from .simplex import SolverLimits, solve
from .workloads import gen_random_lps
from ._native import NativeError, NativeUnavailable

__all__ = [
    "BoxArrays", "BoxLP", "BoxSolution", "InvalidBox", "box_batch_arrays", "solve_box", "solve_box_batch",
    "BatchArrays", "BatchConfig", "BatchReport", "BatchTooLarge", "ChunkPlan", "HeterogeneousBatch",
    "NativeError", "NativeUnavailable", "REFERENCE_GPU_BLOCK_COLS", "SolveOutcome", "SolverLimits",
    "StandardFormLP", "Status", "batch_solve", "batch_solve_arrays", "gen_random_lps", "lp_memory_bytes",
    "plan_chunks", "solve", "standard_form", "support_batch", "validate",
    "GeneralBatch", "GeneralLP", "InfeasibleBounds", "MpsModel", "ParseError", "Relation", "Sense",
    "UnsupportedFeature", "VariableMap", "batch_solve_general", "lower_to_general", "parse_mps",
    "recover_batch", "solve_general", "standardize", "standardize_batch",
    "ORACLE_TOL", "Certificate", "CertificateBatch", "certify_batch", "check_certificate",
]

__version__ = "0.1.0"
