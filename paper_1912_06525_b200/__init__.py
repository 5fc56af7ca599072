"""B200-native Katz query hot path with the API of the reference ``lrckatz``.

Drop-in for the query side of lrckatz (reference __init__.py:9-72): load a
KLRC index built by the reference and answer ``query`` (LRC-Katz Schur
PCG), ``query_cg_baseline`` (plain CG), ``katz_rank`` and ``sparse_katz``
on one GPU through libkatzb200.so (hand-written sm_100a kernels).  Batched
variants (``*_batch``) solve many queries per device call; the recall
harness (``temporal_split``, ``evaluate_recall[_sweep]``) runs on the
batched rankers and graph ingestion (``from_edges``, components) has a
device path.  ``build_index`` builds a KLRC index on the device (native
partitioner, cuSOLVER separator factor, device Lanczos; build.py) for
graphs whose CPU build is out of reach.  The CLI of the reference is out of
scope.
"""

from .eigen import EigenIndex
from .factor_ops import (
    apply_approx_schur_inverse,
    apply_correction,
    block_cholesky,
    build_blocks,
    check_partition,
    dense_cholesky,
)
from .build import (
    DisconnectedGraphError,
    PartitionConfig,
    build_index,
    lanczos_topk,
    partition_vertex_separator,
)

from .evaluate import (
    EmptyPositivesError,
    LinkPredDataset,
    RecallStat,
    evaluate_recall,
    evaluate_recall_sweep,
    temporal_split,
)
from .factor import (
    BlockCholesky,
    DenseCholesky,
    FactorizationError,
    LowRankCorrection,
    SpectrumError,
)
from .graph import (
    ConvergenceError,
    DeviceOperator,
    Graph,
    GraphParseError,
    InadmissibleAlphaError,
    KatzParams,
    from_edges,
    from_edges_device,
    hardest_alpha,
    largest_connected_component,
    largest_connected_component_device,
    load_edge_list,
    spectral_norm,
)
from .index import (
    FORMAT_VERSION,
    BlockPartition,
    GraphIndex,
    IndexChecksumError,
    IndexFormatError,
    IndexMagicError,
    IndexVersionError,
    KatzIndex,
    load_index,
    save_index,
)
from .linkpred import (
    RankedPrediction,
    katz_rank,
    katz_rank_batch,
    pearson,
    sparse_katz,
    sparse_katz_batch,
    topk_device,
)
from .solver import (
    KatzOperator,
    KatzVector,
    SolveReport,
    UnknownNodeError,
    apply_schur,
    cg,
    lrc_pcg,
    query,
    query_batch,
    query_cg_baseline,
    query_cg_baseline_batch,
    schur_rhs,
)

__version__ = "0.1.0"
