"""B200-native training step of multi-GPU isosurface Gaussian splatting
(arxiv 2509.05216), a drop-in for the hot path of the reference package
`isosplat` (project -> sort/bin -> raster fwd -> L1+D-SSIM -> raster bwd ->
ordered reduce -> chain -> Adam, sharded over GPUs).

All compute runs in hand-written sm_100a kernels behind the C ABI of
include/isogs.h (libisogs.so, loaded by _lib.py); there is no CPU fallback.
"""

from .camera import Camera, OrbitSpec, look_at, make_orbit
from .densify import DensifyMapping, densify_and_prune
from .gaussians import (PARAM_NAMES, GaussianCloud, cloud_from_points, load_checkpoint,
                        load_train_state, save_checkpoint, save_train_state, to_device_cloud)
from .metrics import loss_l1_dssim, psnr, quantize8, ssim
from .optim import adam_init, adam_step, position_lr
from .rasterizer import (ParamGradients, ProjectedSplat, RenderAux, SplatBatch,
                         backward_on_tiles, build_tile_lists, chain_to_params,
                         forward_on_tiles, project, reduce_scratch, render_backward,
                         render_forward, sort_order)
from .training import (EvalRecord, PointCloud, TrainConfig, TrainDataset, TrainReport,
                       TrainStats, build_schedule, deterministic_equal)

__version__ = "0.1.0"


def run_training(*args, **kwargs):
    from .engine import run_training as _rt
    return _rt(*args, **kwargs)


def train_single(*args, **kwargs):
    from .engine import train_single as _ts
    return _ts(*args, **kwargs)


def train_distributed(dataset, config, workers: int, **kwargs):
    from .engine import run_training as _rt
    return _rt(dataset, config, workers=workers, **kwargs)
