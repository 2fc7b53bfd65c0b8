"""Eager training steps on 1 GPU for ncu (no CUDA graph, random inputs): `--steps` eager steps.

    ncu --clock-control base -k regex:gemm_kernel --launch-skip 41 --launch-count 41 \
        --metrics gpu__time_duration.sum --csv python tools/ncu_step.py --steps 2
"""
import argparse, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import bench
from paper_2507_05753_b200 import Communicator, ModelConfig, MpContext, WeatherMixerModel
from paper_2507_05753_b200.engine import TrainStep

ap = argparse.ArgumentParser()
ap.add_argument("--steps", type=int, default=2)
ap.add_argument("--config", default="C4")
a = ap.parse_args()
comm = Communicator.from_env()
ctx = MpContext(comm, list(range(comm.world_size)))
cfg_kw, lat_real, vars_real, _ = bench.CONFIGS[a.config]
model = WeatherMixerModel(ctx, ModelConfig(**cfg_kw), init="fast", lat_real=lat_real, vars_real=vars_real)
step = TrainStep(model, graph=False)
bench.fill_random_inputs(step, lat_real, 1234)
for _ in range(a.steps):
    step.run_device()
torch.cuda.synchronize()
print("done", float(step.ws.loss.item()))
