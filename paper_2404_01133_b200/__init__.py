"""B200-native CityGaussian rendering hot path (arXiv 2404.01133).

Drop-in for the render/LoD API of the reference package ``citysplat``:
block-wise LoD selection + aggregation and 3DGS tile rasterization (EWA
projection, tile binning, stable depth sort, front-to-back blending) run as
hand-written sm_100a CUDA kernels in libcsgpu.so, reached through the C ABI in
include/cs_api.h.  There is no CPU fallback: the package refuses to import
when the library has not been built.
"""

from . import _lib

_lib.load()  # fail loudly without the CUDA extension

from .core import CameraView, Gaussian, GaussianCloud, Image  # noqa: E402
from .lod import (AssembledSet, LodScene, VisibilityDecision, assemble_render_set,  # noqa: E402
                  block_visible, build_lod, compress, decide_visibility, mad_bounds, select_level,
                  significance_scores)
from .render import (FrameStats, RenderSettings, SplatPrimitive, project_gaussian,  # noqa: E402
                     rasterize, rasterize_stats, render)
from .service import RenderService  # noqa: E402

__version__ = "0.1.0"
__all__ = [
    "CameraView", "Gaussian", "GaussianCloud", "Image", "LodScene", "VisibilityDecision",
    "AssembledSet", "assemble_render_set", "block_visible", "decide_visibility", "select_level",
    "significance_scores", "compress", "mad_bounds", "build_lod",
    "FrameStats", "RenderSettings", "SplatPrimitive", "project_gaussian", "rasterize",
    "rasterize_stats", "render", "RenderService",
]
