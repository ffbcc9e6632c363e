"""B200-native cover-edge triangle counting (arXiv 2403.02997).

Drop-in for the reference package ``tricount``'s cover-edge path: the same
entry points (``normalize``, ``degree_order``, ``bfs_label``, ``cover_edges``,
``tc_cetc``, ``tc_cetc_sm``, every ``CETC*`` registry entry), backed by
hand-written sm_100a kernels behind the C ABI in include/tricount_b200.h.
There is no CPU fallback: compute calls raise without the CUDA library/GPU.
"""
from .graph import (
    DeviceGraph,
    EdgeList,
    degree_order,
    degree_order_device,
    Graph,
    ParseError,
    device_graph,
    load_edge_list,
    normalize,
    normalize_device,
    parse_edge_list,
    to_edge_list,
)
from .rmat import RmatParams, generate_rmat, rmat_pairs_device
from .bfs import (
    BfsLabeling,
    CoverEdgeSet,
    EdgeClass,
    bfs_label,
    cover_edges,
    enumerate_triangles,
    verify_cover,
)
from .sequential import (
    COVER_RATIO_THRESHOLD,
    SEQUENTIAL_IDS,
    count_sequential,
    tc_cetc,
    tc_cetc_degree,
    tc_cetc_fe,
    tc_cetc_split,
    tc_cetc_split_degree,
    tc_cetc_split_recursive,
    tc_forward_gpu,
)
from .parallel import PARALLEL_IDS, ParallelConfig, tc_cetc_sm, tc_par
from .ops import CetcResult, cetc, cetc_host, cetc_shard
from . import ops
from . import dist
from . import dm
from .dm import DmSimResult, Partition, Shipment, partition_graph, simulate_cetc_dm
from .dm import (CommReport, ScalingFit, comm_report, comm_volume_breakdown, comm_volume_cetc_dm,
                 comm_volume_previous, fit_scaling, format_volume, projected_comm_volume,
                 reports_to_csv, wedge_count)
from . import configs

__version__ = "0.1.0"
