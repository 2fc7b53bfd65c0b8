"""A/B of the GEMM output-tile width on the launches of one eager training step: every launch
with n > 128 runs with the per-shape choice (auto) and forced to 128- and 256-wide tiles,
alternating over rounds (best of rounds per launch). Prints per launch the tile and wave counts
and the three times, then the totals (rank 0; under torchrun the Jigsaw per-rank shapes).

    python tools/tile_n_probe.py                      # 1 GPU
    torchrun --nproc-per-node 4 tools/tile_n_probe.py # Jigsaw 2x2
"""
import math, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import torch.distributed as dist
import bench
from paper_2507_05753_b200 import Communicator, ModelConfig, MpContext, WeatherMixerModel
from paper_2507_05753_b200 import _lib, tensor as T
from paper_2507_05753_b200.engine import TrainStep

comm = Communicator.from_env()
ctx = MpContext(comm, list(range(comm.world_size)))
cfg_kw, lat_real, vars_real, _ = bench.CONFIGS[os.environ.get("CFG", "C4")]
model = WeatherMixerModel(ctx, ModelConfig(**cfg_kw), init="fast", lat_real=lat_real, vars_real=vars_real)
step = TrainStep(model, batch=int(os.environ.get("B", "1")), graph=False)
bench.fill_random_inputs(step, lat_real, 1234 + ctx.pos)
orig = T.gemm_into
shapes, choice = [], [0]


def rec(out, a, b, am, bm, m, n, k, batch=1, *args, **kw):
    if T.GEMM_TIMER is not None and len(shapes) < len(T.GEMM_TIMER) + 1:
        shapes.append((m, n, k, 1 if kw.get("reduce_batch") else batch, am, bm))
    T.GEMM_TILE_N = choice[0] if n > 128 else 0
    try:
        return orig(out, a, b, am, bm, m, n, k, batch, *args, **kw)
    finally:
        T.GEMM_TILE_N = 0


T.gemm_into = rec
for _ in range(3):
    step._body()
torch.cuda.synchronize()
best = {}
for rnd in range(int(os.environ.get("ROUNDS", "3"))):
    for c in (0, 128, 256):
        choice[0] = c
        step._body()  # warm the variant
        torch.cuda.synchronize()
        T.GEMM_TIMER = []
        step._body()
        torch.cuda.synchronize()
        recs, T.GEMM_TIMER = T.GEMM_TIMER, None
        ms = [a.elapsed_time(b) for a, b, _, _ in recs]
        best[c] = ms if c not in best else [min(x, y) for x, y in zip(best[c], ms)]
        if rnd == 0 and c == 0:
            flops = [f for _, _, f, _ in recs]
if comm.rank == 0:
    print(f"{'m':>6} {'n':>6} {'k':>6} {'b':>3} ab  tiles256 waves  tiles128 waves   auto ms  t128 ms  t256 ms  best")
    tot = {c: 0.0 for c in best}
    for i, (m, n, k, bt, am, bm) in enumerate(shapes[:len(flops)]):
        cg = 2 if m > 128 else 1
        t256 = math.ceil(m / (128 * cg)) * math.ceil(n / 256) * bt
        t128 = math.ceil(m / (128 * cg)) * math.ceil(n / 128) * bt
        u = _lib.num_sms() // cg
        row = {c: best[c][i] for c in best}
        for c in best:
            tot[c] += row[c]
        win = min(row, key=row.get)
        print(f"{m:6d} {n:6d} {k:6d} {bt:3d} {am}{bm} {t256:8d} {t256 / u:5.2f} {t128:8d} {t128 / u:5.2f} "
              f"{row[0]:9.3f} {row[128]:8.3f} {row[256]:8.3f}  {win if win else 'auto'}")
    print("total ms: " + "  ".join(f"{('auto' if c == 0 else c)} {v:.3f}" for c, v in tot.items())
          + f"  (best per launch {sum(min(best[c][i] for c in best) for i in range(len(flops))):.3f})")
if comm.world_size > 1:
    dist.barrier()
os._exit(0)
