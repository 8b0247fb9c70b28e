"""B200-native MPDATA / neighbour-stencil hot path of arXiv 1908.06094.

Drop-in for the hot path of the reference package ``tristencil`` (the
MPDATA transport step, the 9-relation neighbour reductions, the Table-1
indexing kernels and the field layout/numbering machinery they need).  The
public names below mirror ``tristencil``'s; compute runs in hand-written
sm_100a CUDA kernels in ``libtsg.so`` behind the C ABI of include/tsg.h.
PyTorch supplies device memory and streams only.  There is no CPU fallback.
"""

from .topology import LocationType, PatchSpec, element_count, element_coord, element_id
from .layouts import (
    AXES,
    DEFAULT_DIM_ORDER,
    AccessMethod,
    LayoutSpec,
    LinearLayout,
    Numbering,
    Permutation,
    check_access_combo,
    coalescing_fraction,
    direct_sweep_groups,
    hilbert_rank,
    hilbert_xy,
    make_permutation,
    sn_offset,
)
from .connectivity import (
    OFFSET_TABLES,
    NeighborTable,
    StructuredOffsets,
    build_neighbor_table,
    dump_tables,
    edge_signs_table,
    neighbor_len,
    structured_offsets,
)
from .stencil import CompositionError
from .storage import (
    DivergenceError,
    Field,
    FieldMeta,
    Selector,
    StalenessError,
    StorageError,
    make_storage,
    plane_access_total,
    reset_counters,
    sync,
)
from .executors import (
    RunStats,
    TileSpec,
    TimingResult,
    halo_update,
    run_fused,
    run_gpu,
    run_time_loop,
    run_naive,
    time_computation,
)
from .mpdata import (
    GeometryFields,
    MpdataParams,
    StateFields,
    build_divergence,
    build_geometry,
    build_mpdata,
    build_state,
    init_preset,
    load_field_csv,
    total_mass,
)
from .kernels import (
    build_kernel,
    build_reduce,
    field_to_flat,
    flat_to_field,
    gather_groups,
    make_kernel_fields,
    run_neighbor_sum,
    run_neighbor_sum_scaled,
    unpermute,
)
from .flat import StructuredStepper, transport_step, transport_step_structured
from .traffic import TrafficReport, TrafficRow
from . import reference  # the flat stage API of tristencil.reference

UNFUSED_PLANE_WEIGHTS = {"nodes": (7, 3), "edges": (1, 1)}  # bench.py:57-60
FUSED_PLANE_WEIGHTS = {"nodes": (4, 1)}

__version__ = "0.1.0"
