"""paper_2604_04696_b200 — B200-native GPIR server pipeline (arXiv 2604.04696).

Drop-in for the reference `latpir` server path: `encode_database`,
`answer_batch` / `respond` (aliases `process_batch` / `process_query`), with
the reference's value types and planner API.  All server computation runs in
libgpir.so (hand-written sm_100a CUDA, include/gpir.h); there is no CPU
fallback.
"""
from .errors import InvalidArgument, InvalidConfig, InvalidState, NativeError, ParseError, PirError
from .planner import ExecMode, ExecutionPlan, HardwareModel, Phase, build_plan
from .protocol import (
    Context,
    EncodedDatabase,
    ServeStats,
    answer_batch,
    encode_database,
    encode_database_array,
    encode_database_device,
    get_context,
    process_batch,
    process_query,
    respond,
    upload_database,
)
from .values import (
    BfvCiphertext,
    ClientKeys,
    ClientQuery,
    DbConfig,
    Domain,
    EvalKey,
    GadgetConfig,
    HeParams,
    LayoutKind,
    Modulus,
    Response,
    RgswCiphertext,
    RnsBasis,
    RnsPoly,
    ct_from_raw,
    default_basis,
    default_params,
    test_params,
)

__all__ = [
    "BfvCiphertext", "ClientKeys", "ClientQuery", "Context", "DbConfig", "Domain", "EncodedDatabase", "EvalKey",
    "ExecMode", "ExecutionPlan", "GadgetConfig", "HardwareModel", "HeParams", "InvalidArgument", "InvalidConfig",
    "InvalidState", "LayoutKind", "Modulus", "NativeError", "ParseError", "Phase", "PirError", "Response",
    "RgswCiphertext", "RnsBasis", "RnsPoly", "ServeStats", "answer_batch", "build_plan", "ct_from_raw",
    "default_basis", "default_params", "encode_database", "encode_database_array", "encode_database_device",
    "get_context", "process_batch",
    "process_query", "respond", "test_params", "upload_database",
]

__version__ = "0.1.0"
