"""B200-native (sm_100a) WeatherMixer training step under Jigsaw parallelism (arXiv 2507.05753).

Drop-in for the reference `jigsaw` package's hot path: same names as its __init__.py
(ModelConfig, WeatherMixerModel, MpContext, pnt/pnn/ptn, comm_volume, ShardSpec, shard,
gather, MatmulMode, ProcessGroup), executed by hand-written tcgen05/TMA kernels in
libjigsaw_sm100.so and NCCL / NVLink peer memory. The training loop around the step
(engine.TrainStep / Trainer, train.AdamConfig with the SPEC schedule and clipping,
data.TileLoader, checkpoint.save / load) follows the reference SPEC's train module.
"""
from .comm import Communicator, ProcessGroup
from .config import ModelConfig
from .errors import CommError, CommTimeout, ConfigError, ShapeError, WorkerError
from .model import Layout, WeatherMixerModel
from .layers import MixerBlock, ShardedLayerNorm, ShardedLinear
from .params import Param
from .parallel import MpContext, comm_volume, pnn, pnt, ptn
from .sharding import ShardSpec, gather, shard
from .tensor import MatmulMode
from .train import AdamConfig
from .data import TileLoader
from .engine import Trainer, TrainStep
from . import checkpoint

__all__ = [
    "MixerBlock", "Param", "ShardedLayerNorm", "ShardedLinear",
    "Communicator", "CommError", "CommTimeout", "ConfigError", "Layout", "MatmulMode", "ModelConfig",
    "MpContext", "ProcessGroup", "ShapeError", "ShardSpec", "WeatherMixerModel", "WorkerError",
    "comm_volume", "gather", "pnn", "pnt", "ptn", "shard",
    "AdamConfig", "TileLoader", "TrainStep", "Trainer", "checkpoint",
]
