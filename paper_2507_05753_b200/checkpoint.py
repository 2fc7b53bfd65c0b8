"""Per-rank sharded checkpoints of a training step.

One file per model-parallel position, shards never merged:

    <dir>/shard-<pos>-of-<n>.jgck
      line 1   JSON header {"format": "jigsaw-ckpt", "version": 1, "rank": pos, "n": n,
               "grid": [R, C], "config_hash": ..., "op_dtype": ..., "step": t, "records": k}
      then k records, little-endian:
               u32 name length, name (utf-8), u32 dtype length, numpy dtype str ("<f4", "<i4"),
               u32 ndim, ndim x u64 dims, payload (C order)

Records: param/<name> (fp32 master), adam_m/<name>, adam_v/<name>, step (int32 Adam counter =
schedule position). A Trainer checkpoint adds a "trainer" header entry: the epoch, the batches of
it already trained and the rollout RNG's epoch-start state, so a resumed fine-tuning run draws
the same rollouts and samples as the uninterrupted one. Loading checks format, world shape and model-config hash and restores
bit-identical parameters, moments and step; the bf16 operand copies are re-derived. Within a
data-parallel group every replica holds the same shard, so only dp index 0 writes.
"""
from __future__ import annotations

import json
import os
import struct

import numpy as np
import torch

from .errors import ConfigError

FORMAT, VERSION = "jigsaw-ckpt", 1


def shard_path(directory: str, pos: int, n: int) -> str:
    return os.path.join(directory, f"shard-{pos}-of-{n}.jgck")


def _records(step) -> list[tuple[str, np.ndarray]]:
    m, f = step.model, step.model.flat
    out = []
    for name, p in m.params.items():
        out.append((f"param/{name}", p.data))
        out.append((f"adam_m/{name}", f.view(name, f.m)))
        out.append((f"adam_v/{name}", f.view(name, f.v)))
    out.append(("step", step.step_count))
    return [(k, t.detach().cpu().numpy()) for k, t in out]


def _header(step, nrec: int, extra: dict | None = None) -> dict:
    m = step.model
    h = {"format": FORMAT, "version": VERSION, "rank": m.ctx.pos, "n": m.ctx.n, "grid": [m.R, m.C],
         "config_hash": m.cfg.content_hash(), "op_dtype": str(m.op_dtype).replace("torch.", ""),
         "step": int(step.step_count.item()), "records": nrec}
    h.update(extra or {})
    return h


def save(step, directory: str, extra: dict | None = None) -> str | None:
    """Write this rank's shard (TrainStep state: master weights, Adam moments, step counter; `extra`
    header fields, e.g. the Trainer's epoch / position / rollout-RNG state). Returns the file
    written, or None on dp replicas other than index 0."""
    if step.model.ctx.dp_index != 0:
        return None
    if step.model.device.type == "cuda":
        torch.cuda.synchronize()
    os.makedirs(directory, exist_ok=True)
    recs = _records(step)
    path = shard_path(directory, step.model.ctx.pos, step.model.ctx.n)
    tmp = path + ".tmp"
    with open(tmp, "wb") as fh:
        fh.write((json.dumps(_header(step, len(recs), extra), sort_keys=True) + "\n").encode())
        for name, a in recs:
            a = np.ascontiguousarray(a)
            dt = a.dtype.newbyteorder("<")
            nb, db = name.encode(), dt.str.encode()
            fh.write(struct.pack("<I", len(nb)) + nb + struct.pack("<I", len(db)) + db)
            fh.write(struct.pack("<I", a.ndim) + struct.pack(f"<{a.ndim}Q", *a.shape))
            fh.write(a.astype(dt, copy=False).tobytes())
    os.replace(tmp, path)
    return path


def read(path: str) -> tuple[dict, dict[str, np.ndarray]]:
    """Parse one shard file -> (header, {record name: array})."""
    with open(path, "rb") as fh:
        header = json.loads(fh.readline().decode())
        if header.get("format") != FORMAT or header.get("version") != VERSION:
            raise ConfigError(f"{path}: not a {FORMAT} v{VERSION} file")
        recs = {}
        for _ in range(header["records"]):
            (nl,) = struct.unpack("<I", fh.read(4))
            name = fh.read(nl).decode()
            (dl,) = struct.unpack("<I", fh.read(4))
            dt = np.dtype(fh.read(dl).decode())
            (nd,) = struct.unpack("<I", fh.read(4))
            shape = struct.unpack(f"<{nd}Q", fh.read(8 * nd)) if nd else ()
            cnt = int(np.prod(shape)) if nd else 1
            recs[name] = np.frombuffer(fh.read(cnt * dt.itemsize), dtype=dt).reshape(shape)
    return header, recs


def load(step, directory: str) -> dict:
    """Restore this rank's shard into a TrainStep built for the same config and world shape."""
    m, f = step.model, step.model.flat
    path = shard_path(directory, m.ctx.pos, m.ctx.n)
    if not os.path.exists(path):
        found = sorted(x for x in os.listdir(directory) if x.endswith(".jgck")) if os.path.isdir(directory) else []
        if found:  # a checkpoint of another world shape
            with open(os.path.join(directory, found[0]), "rb") as fh:
                h = json.loads(fh.readline().decode())
            raise ConfigError(f"checkpoint world shape {h.get('n')}-way {tuple(h.get('grid', ()))} does not match "
                              f"this world's {m.ctx.n}-way {(m.R, m.C)} ({directory})")
        raise ConfigError(f"no shard for position {m.ctx.pos} of a {m.ctx.n}-way world ({m.R}x{m.C}) in "
                          f"{directory}; found {found}")
    header, recs = read(path)
    if header["n"] != m.ctx.n or list(header["grid"]) != [m.R, m.C]:
        raise ConfigError(f"checkpoint world shape {header['n']}-way {tuple(header['grid'])} does not match this "
                          f"world's {m.ctx.n}-way {(m.R, m.C)}")
    if header["rank"] != m.ctx.pos:
        raise ConfigError(f"{path}: shard of position {header['rank']}, expected {m.ctx.pos}")
    if header["config_hash"] != m.cfg.content_hash():
        raise ConfigError(f"checkpoint model config {header['config_hash']} != {m.cfg.content_hash()}")
    for name, p in m.params.items():
        for key, dst in ((f"param/{name}", p.data), (f"adam_m/{name}", f.view(name, f.m)),
                         (f"adam_v/{name}", f.view(name, f.v))):
            a = recs[key]
            if tuple(a.shape) != tuple(dst.shape):
                raise ConfigError(f"{key}: checkpoint shape {a.shape} != local shape {tuple(dst.shape)}")
            dst.copy_(torch.from_numpy(a.copy()))
    step.step_count.copy_(torch.from_numpy(recs["step"].copy()))
    m.sync_operand_copies()
    return header
