"""B200-native VR-NeRF frame renderer (arXiv 2311.02542), drop-in for the reference's
rendering path.  See DESIGN.md.  The CUDA library is required (no CPU fallback)."""
from ._abi import Error  # noqa: F401
from .renderer import (CameraModel, ColorSpaceMode, ContractionMode, DeviceModel,  # noqa: F401
                       FieldConfig, HashGridConfig, Image, OccupancyGrid, RadianceField,
                       RenderOptions, RowStats, device_info, load_checkpoint, render_rows,
                       save_checkpoint)
from .scheduler import (FrameStats, RowRange, StatsSummary, WorkerAssignment,  # noqa: F401
                        aggregate_stats, assign_rows, equal_assignment, next_assignment,
                        run_frame)

__version__ = "0.1.0"
