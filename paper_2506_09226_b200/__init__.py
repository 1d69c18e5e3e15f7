"""B200-native drop-in for the ``shufflecast`` relational hot path.

Same public names as the reference package (`/root/reference/pkg/src/
shufflecast/__init__.py:9-72`) for the path in scope:
storage, relational operators, exchange operators, the SPMD engine and the
TPC-H query drivers.  Tables live in HBM; operators run as hand-written
sm_100a kernels in ``libscx.so`` (C-ABI in include/scx.h) -- there is no
CPU fallback.  The reference's analytical models, topology parser, CLI and
virtual-time simulator are out of scope; the in-process
cluster (``create_cluster(topo, MODE_IN_PROCESS)`` + ``run_workers``) runs
N workers as virtual ranks on one GPU.
"""

from .cluster import (MODE_GLOO, MODE_IN_PROCESS, MODE_NCCL, MODE_SIMULATED, Cluster,
                      ClusterConfigError, DeadlockError, Endpoint, GroupOp, ProtocolError, Topology,
                      TopologyError, barrier, create_cluster, run_workers)
from .collectives import all_reduce, broadcast_collective, broadcast_p2p, group_execute
from .data import (DEFAULT_PARTITION_KEYS, DataError, Dataset, PartitionedDataset, generate,
                   partition_dataset)
from .engine import (EXCHANGE_PLANS, DeviceContext, ExchangePlan, PlanError, RunReport,
                     get_plan, load_tables, partition_tables, q12_variants, reference_run,
                     result_digest, run_query)
from .exchange import (ExchangeStats, broadcast_table, hash_keys, hash_partition,
                       shuffle_table, size_exchange)
from .expr import codes_where, isin, where
from .queries import PLAN_FUNCTIONS, SUPPORTED_QUERIES
from .relops import TableView, filter_table, group_aggregate, local_hash_join
from .table import (Column, ColumnTable, HostColumn, HostTable, SchemaError, concat_tables,
                    date32_col, date_to_days, days_to_date, dict_col, dict_col_from_strings,
                    float64_col, int64_col, tables_equal)
from ._lib import ScxError

LocalContext = DeviceContext     # single-GPU context == the reference's single context
WorkerContext = DeviceContext

__version__ = "0.1.0"
