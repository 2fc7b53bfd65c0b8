"""Per-rank NVLink bytes per C4 training step of this schedule for every grid (analytic,
jigsaw_grid.step_exchange_bytes on a stand-in model object: no GPU, no process group), with the
comm roofline at the measured 770 GB/s and the GEMM time at the sustained bf16 peak.

    python tools/comm_table.py
"""
import json
import os
import sys
from types import SimpleNamespace

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2507_05753_b200.config import ModelConfig  # noqa: E402
from paper_2507_05753_b200.jigsaw_grid import step_exchange_bytes  # noqa: E402

C4 = ModelConfig(n_vars=70, grid=(728, 1440), patch=(8, 8), d_emb=4320, d_tok=8640, d_ch=4320, n_blocks=3)
peak = json.load(open(os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "MEASURED_PEAKS.json")))
sustained = peak.get("bf16_tflops_sustained", 1392.2)


def stub(R, C):
    cfg = C4
    E, H, F, Kd, T, V = cfg.d_emb, cfg.d_ch, cfg.patch_features, cfg.d_tok, cfg.tokens, cfg.n_vars
    nb = cfg.n_blocks
    encdec_col = E // C + F // C + V // C
    body_col = nb * (4 * E // C + Kd // C + H // C + E // C)
    body_row = nb * (T // R)
    kr = {("encdec", "vec_col"): (0, encdec_col), ("encdec", "vec_row"): (0, 0),
          ("body", "vec_col"): (0, body_col), ("body", "vec_row"): (0, body_row)}
    flat = SimpleNamespace(CLASSES=("encdec", "body"), kind_range=kr)
    m = SimpleNamespace(cfg=cfg, R=R, C=C, ctx=SimpleNamespace(n=R * C), op_dtype=torch.bfloat16, flat=flat,
                        _ws=SimpleNamespace(grid=SimpleNamespace(peer_moments=C > 1)))
    return m


rows = []
for R, C in ((1, 2), (2, 1), (2, 2), (4, 1), (4, 2), (8, 1)):
    m = stub(R, C)
    v = step_exchange_bytes(m, 1, 1)
    n = R * C
    fl = 3 * (4 * C4.tokens * C4.patch_features * C4.d_emb + C4.n_blocks * 4 * C4.tokens * C4.d_emb
              * (C4.d_tok + C4.d_ch)) - 2 * C4.tokens * C4.patch_features * C4.d_emb
    t_comm = v["total"] / 770e9 * 1e3
    t_gemm = fl / n / (sustained * 1e12) * 1e3
    rows.append((f"{R}x{C}", v["total"], t_comm, t_gemm))
print("| grid | NVLink bytes / rank / step | t_comm at 770 GB/s (ms) | t_gemm at sustained peak (ms) | comm / gemm |")
print("|---|---|---|---|---|")
for g, b, tc, tg in rows:
    print(f"| {g} | {b / 1e9:.2f} GB | {tc:.2f} | {tg:.2f} | {tc / tg:.2f} |")
