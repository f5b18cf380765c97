"""B200-native DisCo candidate scoring: the fused-op estimator and the
iteration simulator on sm_100a, behind the reference ``fuseopt`` package's
estimator / simulator / search entry points.

The CUDA library (paper_2209_12769_b200/_build/libdiscob200.so) is required:
every device entry point raises if it is missing; there is no CPU fallback.
"""

from .comm import CommModelParams, load_params, predict, save_params
from .errors import (
    CycleError,
    DeviceError,
    DimensionMismatch,
    FuseoptError,
    GraphFormatError,
    InvalidConfig,
    LimitExceeded,
    MissingCost,
    NotNeighbors,
    UnknownOp,
)
from .estimator import (
    DeviceCostProviders,
    EstimatorModel,
    EstimatorVariant,
    Profile,
    analytic_model,
    load_model,
    load_profile,
    lookup,
    make_cost_providers,
    predict_fused_groups,
)
from .features import SubgraphFeatures, featurize, group_io, predict_fused
from .graph import (
    AllReduceInstr,
    DataEdge,
    FusionGroup,
    GraphMeta,
    HloGraph,
    ModuleStats,
    OpNode,
    TensorBucket,
    build_graph,
    canonical_hash,
    graph_from_doc,
    graph_to_doc,
    load_graph,
    module_stats,
    save_graph,
    with_fusion_state,
)
from .rewrite import (
    OptimizationMethod,
    RewriteOutcome,
    bucket_pairs,
    fuse_allreduce,
    fuse_dup,
    fuse_nondup,
    fusible_pairs,
    make_candidates,
    neighbors_allreduce,
    random_apply,
)
from .search import (
    LockstepSearch,
    SearchConfig,
    SearchResult,
    TraceRecord,
    backtracking_search,
    exhaustive_search,
    greedy_postorder_fusion,
    topo_order,
    lockstep_search,
    threshold_allreduce_fusion,
)
from .simulator import CostProviders, Timeline, cost, cost_batch, fo_bound, format_timeline, report_lines, simulate
from .workloads import HardwareParams, load_workload, oracle_providers, oracle_time

__version__ = "0.1.0"
