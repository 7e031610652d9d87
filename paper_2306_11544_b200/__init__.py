"""B200-native implementation of the cellbench hot path (arXiv 2306.11544).

The public names mirror the reference package ``cellbench``'s hot-path API
(core / diffusion / mechanics / parallel / errors), so a caller can switch
``import cellbench as cb`` to ``import paper_2306_11544_b200 as cb`` for the
per-step loop.  All compute runs in libcellgpu.so (sm_100a CUDA kernels
behind the C-ABI of include/cellgpu.h); there is no CPU fallback.
"""

from .core import (
    POSITION_EPS,
    CartesianMesh,
    Cell,
    CellContainer,
    Microenvironment,
    Vec3,
    rebin_cells,
    sort_cells_by_voxel,
    vec3,
    voxel_of,
)
from .diffusion import (TraversalMode, apply_cell_exchange, compute_gradients, lod_step,
                        refresh_nonempty_list)
from .errors import (
    CapacityError,
    CellBenchError,
    ConfigError,
    ContainerStateError,
    DeviceError,
    DomainError,
    NumericError,
)
from .mechanics import (
    EPS_SKIP,
    AllocationMode,
    InteractionParams,
    MechanicsSchedule,
    ScheduleKind,
    check_binning_exact,
    integrate_positions,
    pair_velocity_contribution,
    update_velocities,
)
from .parallel import RegionRecord, WorkerPool, WorkerStats, static_ranges
from .population import DEFAULT_CELL_CAP, attempt_divisions, division_draws
from .checksum import state_checksum

__version__ = "0.1.0"


def __getattr__(name):
    # Heavy/optional pieces load lazily (they need torch + CUDA).
    if name == "Simulation":
        from .engine import Simulation

        return Simulation
    if name in ("CONFIGS", "SimConfig", "make_inputs"):
        from . import configs

        return getattr(configs, name)
    raise AttributeError(name)
