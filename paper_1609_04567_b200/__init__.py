"""B200-native loop-of-stencil-reduce (arxiv 1609.04567), drop-in for `stencilkit`.

Same pattern vocabulary as the reference package (stencilkit/__init__.py):
grids, elemental functions, combinators, the four loop variants,
partitioned loops and stream composition.  Underneath, every stencil sweep
is a hand-written sm_100a kernel fused with its reduce and loop test; the
loop runs on the GPU.
"""

from .grid import (ABSENT, Grid, GridError, IndexedNeighborhood, Neighborhood, grid_get_padded,
                   grid_new, indexed_neighborhood_at, is_absent, neighborhood_at)
from .ledger import CopyLedger
from .loop import (Condition, DeviceCond, LoopReport, LoopState, loop_stencil_reduce,
                   loop_stencil_reduce_d, loop_stencil_reduce_i, loop_stencil_reduce_s,
                   stop_after)
from .loop import SequentialExecutor
from .partition import (BlockInfo, DeploymentMode, DeviceExecutor, DeviceRows, ParallelExecutor,
                        Partition, PartitionSet,
                        WorkerGroup, halo_exchange, model_ledger, parallel_loop, parallel_step,
                        partition)
from .patterns import (Combinator, Delta, DeviceKernel, DeviceUnsupported, ElementalFn,
                       StencilError, abs_change, apply_to_all, map_pattern, max_combinator,
                       reduce_all, reduce_pattern, sq_change, stencil_apply,
                       stencil_apply_indexed, sum_combinator)

from .jit import CudaCombine, CudaDelta, cuda_elemental
from .pgm import PgmError, read_pgm, write_pgm
from .streams import (OrderedFarm, Pipeline, Stage, StreamError, StreamReport, ordered_farm,
                      pipeline, run_stream)

__version__ = "0.1.0"
