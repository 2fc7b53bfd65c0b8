"""CLI on the GPU: `verify` (sharded model vs the reference's golden results) at n = 1 / 2 and
`train` (Trainer over synthetic samples: loss CSV + checkpoint shards)."""
from __future__ import annotations

import json
import os
import subprocess
import sys

import pytest
import torch

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
DESK = {"n_vars": 8, "grid": [32, 64], "patch": [4, 4], "d_emb": 64, "d_tok": 128, "d_ch": 64, "n_blocks": 2}


def _cfg(tmp_path, **kw):
    p = tmp_path / "exp.json"
    p.write_text(json.dumps({"model": DESK, **kw}))
    return str(p)


@pytest.mark.parametrize("n", [1, 2])
def test_cli_verify(tmp_path, n):
    if not torch.cuda.is_available() or torch.cuda.device_count() < n:
        pytest.skip(f"needs {n} GPUs")
    cfg = _cfg(tmp_path, world={"n_way": n})
    cmd = [sys.executable, "-m", "paper_2507_05753_b200", "verify", "--config", cfg, "--out", str(tmp_path)]
    if n > 1:
        cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={n}",
               "--master-addr=127.0.0.1", "--master-port=29577", "-m", "paper_2507_05753_b200", *cmd[3:]]
    p = subprocess.run(cmd, capture_output=True, text=True, cwd=ROOT, timeout=600)
    assert p.returncode == 0, p.stdout[-2000:] + p.stderr[-3000:]
    rep = json.load(open(tmp_path / "verify.json"))
    assert all(c["pass"] for c in rep["checks"].values()), rep


def test_cli_train(tmp_path):
    if not torch.cuda.is_available():
        pytest.skip("needs a GPU")
    cfg = _cfg(tmp_path, train={"steps": 4, "warmup_steps": 1, "total_steps": 4, "clip_norm": 1.0},
               data={"synthetic": 6}, dtype="bf16")
    out = tmp_path / "run"
    p = subprocess.run([sys.executable, "-m", "paper_2507_05753_b200", "train", "--config", cfg, "--out", str(out)],
                       capture_output=True, text=True, cwd=ROOT, timeout=600)
    assert p.returncode == 0, p.stdout[-2000:] + p.stderr[-3000:]
    lines = (out / "loss.csv").read_text().strip().splitlines()
    assert len(lines) == 5 and lines[0].startswith("epoch,step")
    assert os.listdir(out / "ckpt")
