"""B200-native spatially partitioned 3D U-Net training (arXiv 1909.03108).

Drop-in for the reference ``voxmesh`` API on the hot path (mesh / layout,
shard / gather, halo exchange, halo-exchanging conv3d, U-Net builder, loss,
train step), with every kernel hand-written for sm_100a behind the C ABI of
``libvoxmesh_sm100.so`` (include/vm_api.h).
"""

from .errors import (
    GraphBuildError,
    HaloError,
    ShardingError,
    VoxmeshError,
    WorkerFailed,
)
from .mesh import DeviceMesh, WorkerContext, create_mesh
from .sharding import Layout, ShardedTensor, TensorSpec, gather, shard
from .halo import HaloSpec, PaddedBlock, exchange_byte_count, halo_exchange, halo_exchange_backward
from .unet import LayerGraph, UNetConfig, build, init_params, recipe_for_resolution
from .ops import (
    ConvParams,
    ConvTape,
    concat_channels,
    conv3d_backward,
    conv3d_forward,
    maxpool2_backward,
    maxpool2_forward,
    relu,
    relu_backward,
    softmax_channels,
    upsample2_backward,
    upsample2_forward,
)
from .training import (
    BatchSource,
    combined_loss,
    cross_entropy_loss,
    one_hot,
    soft_dice_loss,
    LossWeights,
    TrainConfig,
    TrainState,
    dice_global,
    dice_per_case,
    evaluate,
    hard_dice,
    install_params,
    load_checkpoint,
    save_checkpoint,
    train_loop,
)

__version__ = "0.1.0"

__all__ = [
    "DeviceMesh",
    "GraphBuildError",
    "HaloError",
    "HaloSpec",
    "LayerGraph",
    "Layout",
    "PaddedBlock",
    "ShardedTensor",
    "ShardingError",
    "TensorSpec",
    "UNetConfig",
    "VoxmeshError",
    "WorkerContext",
    "WorkerFailed",
    "build",
    "create_mesh",
    "exchange_byte_count",
    "gather",
    "halo_exchange",
    "halo_exchange_backward",
    "init_params",
    "recipe_for_resolution",
    "shard",
    "BatchSource",
    "LossWeights",
    "TrainConfig",
    "TrainState",
    "dice_global",
    "dice_per_case",
    "evaluate",
    "hard_dice",
    "install_params",
    "load_checkpoint",
    "save_checkpoint",
    "train_loop",
    "combined_loss",
    "cross_entropy_loss",
    "one_hot",
    "soft_dice_loss",
    "ConvParams",
    "ConvTape",
    "concat_channels",
    "conv3d_backward",
    "conv3d_forward",
    "maxpool2_backward",
    "maxpool2_forward",
    "relu",
    "relu_backward",
    "softmax_channels",
    "upsample2_backward",
    "upsample2_forward",
]
