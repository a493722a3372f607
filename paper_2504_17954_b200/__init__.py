"""B200-native editable-Gaussian splatting hot path (iVR-GS, arxiv 2504.17954).

Drop-in for the hot path of the reference package ``voxsplat``: the public
names below keep the reference's signatures; the compute runs in the
in-tree CUDA library ``libivrgs.so`` (sm_100a), reached through the C ABI in
``include/ivrgs.h``.  Importing the package does not touch the GPU; the first
kernel call loads the library and fails loudly if it is missing.
"""

from .errors import (  # noqa: F401
    BadMagic, ChecksumMismatch, CorruptIndex, CulledBehindCamera, DatasetEmpty, DivergedLoss,
    EmptyInput, MixedStage, NonFiniteGradient, OutOfRange, ShapeMismatch, UnknownAttribute,
    VersionUnsupported, VoxSplatError,
)
from .gaussians import Camera, GaussianGeometry, ShColor, orbit_camera, project_gaussians  # noqa: F401
from .rasterizer import (  # noqa: F401
    RenderOutput, rasterize_backward, rasterize_forward, render_attribute_map,
)
from .scene import (  # noqa: F401
    BasicSceneModel, ComposedScene, DeviceScene, EditState, EffectiveScene, FrameGraph, FramePipeline,
    apply_edits, compose_device, render_composed,
)
from .shading import (  # noqa: F401
    LightConfig, Palette, ShadingAttributes, shade_backward, shade_gaussians,
)
from .trainer import (  # noqa: F401
    TrainConfig, ViewDataset, render_model, train_base, train_editable,
)
from .vq import Codebook, assign_nearest, dequantize_model, kmeans, quantize_model  # noqa: F401

__version__ = "0.1.0"
