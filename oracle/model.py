"""ORACLE (test infrastructure): numpy restatement of reference model.py / parallel.py for the
WeatherMixer step — config, global init, serial (n=1) forward/backward, per-rank layouts.

Follows:
  ModelConfig / validate          model.py:41-111
  token_sets / contiguous_split   model.py:114-121, sharding.py:24-27
  global init, registration order model.py:312-398 (uniform(+-1/sqrt(fan_in)) drawn in f64)
  Layout.local (n = 2, 4)         model.py:135-150
  forward                         model.py:406-426, MixerBlock.forward model.py:268-282,
                                  ShardedLinear.forward parallel.py:515-526 (n = 1)
  backward                        model.py:428-445, MixerBlock.backward model.py:284-297,
                                  ShardedLinear.backward parallel.py:528-549 (n = 1)
"""
from __future__ import annotations

import hashlib
from dataclasses import dataclass

import numpy as np

from . import ops


@dataclass
class Config:
    n_vars: int = 8
    grid: tuple = (32, 64)
    patch: tuple = (4, 4)
    d_emb: int = 64
    d_tok: int = 128
    d_ch: int = 64
    n_blocks: int = 3

    @property
    def patch_grid(self):
        return self.grid[0] // self.patch[0], self.grid[1] // self.patch[1]

    @property
    def tokens(self):
        gl, gw = self.patch_grid
        return gl * gw

    @property
    def patch_features(self):
        return self.patch[0] * self.patch[1] * self.n_vars


# --------------------------------------------------------------------------- axis splits
def token_sets(cfg: Config, parts: int = 2):
    """Strided longitude split of the row-major token axis (model.py:114-121 for parts=2)."""
    gl, gw = cfg.patch_grid
    w = gw // parts
    return [np.array([a * gw + b for a in range(gl) for b in range(i * w, (i + 1) * w)], dtype=np.int64)
            for i in range(parts)]


def contiguous_split(size: int, parts: int):
    """sharding.py:20-27."""
    chunk = -(-size // parts)
    return [np.arange(p * chunk, (p + 1) * chunk) for p in range(parts)]


# --------------------------------------------------------------------------- init
def param_specs(cfg: Config):
    """(name, shape, fan_in or None, kind, row_axis, col_axis, lr_class, const) in the reference's
    registration order (model.py:336-389). Axis names: E, F, T, K (d_tok), H (d_ch), C (vars)."""
    E, F, T, K, H, C = cfg.d_emb, cfg.patch_features, cfg.tokens, cfg.d_tok, cfg.d_ch, cfg.n_vars
    out = [("enc.w", (E, F), F, "matrix", "E", "F", "encdec", None),
           ("enc.b", (E,), None, "vec_col", None, "E", "encdec", 0.0)]
    for i in range(cfg.n_blocks):
        p = f"block{i}."
        out += [
            (p + "ln1.gamma", (E,), None, "vec_col", None, "E", "body", 1.0),
            (p + "ln1.beta", (E,), None, "vec_col", None, "E", "body", 0.0),
            (p + "tok1.w", (T, K), T, "matrix", "T", "K", "body", None),
            (p + "tok1.b", (K,), None, "vec_col", None, "K", "body", 0.0),
            (p + "tok2.w", (T, K), K, "matrix", "T", "K", "body", None),
            (p + "tok2.b", (T,), None, "vec_row", "T", None, "body", 0.0),
            (p + "ln2.gamma", (E,), None, "vec_col", None, "E", "body", 1.0),
            (p + "ln2.beta", (E,), None, "vec_col", None, "E", "body", 0.0),
            (p + "ch1.w", (H, E), E, "matrix", "H", "E", "body", None),
            (p + "ch1.b", (H,), None, "vec_col", None, "H", "body", 0.0),
            (p + "ch2.w", (E, H), H, "matrix", "E", "H", "body", None),
            (p + "ch2.b", (E,), None, "vec_col", None, "E", "body", 0.0),
        ]
    out += [("dec.w", (F, E), E, "matrix", "F", "E", "encdec", None),
            ("dec.b", (F,), None, "vec_col", None, "F", "encdec", 0.0),
            ("blend.w", (C,), None, "vec_col", None, "C", "body", 0.5)]
    return out


def init_params(cfg: Config, seed: int = 0, dtype=np.float64):
    """Global parameters exactly as the reference draws them (model.py:312, 323-334)."""
    rng = np.random.default_rng(seed)
    params = {}
    for name, shape, fan_in, kind, _, _, _, const in param_specs(cfg):
        if fan_in is not None:
            bound = 1.0 / np.sqrt(fan_in)
            params[name] = rng.uniform(-bound, bound, size=shape).astype(dtype)
        else:
            params[name] = np.full(shape, const, dtype=dtype)
    return params


def params_digest(params) -> str:
    h = hashlib.sha256()
    for name in params:
        h.update(name.encode())
        h.update(np.ascontiguousarray(params[name]).tobytes())
    return h.hexdigest()[:16]


# --------------------------------------------------------------------------- layouts
def axis_sets(cfg: Config, axis: str, parts: int):
    if axis == "T":
        return token_sets(cfg, parts)
    size = {"E": cfg.d_emb, "F": cfg.patch_features, "K": cfg.d_tok, "H": cfg.d_ch, "C": cfg.n_vars}[axis]
    return contiguous_split(size, parts)


def local_tile(cfg: Config, name: str, glob: np.ndarray, R: int, C: int, r: int, c: int) -> np.ndarray:
    """Rank (r, c)'s tile of a global parameter on an R x C Jigsaw grid (SURVEY 8e tile maps).

    Matrices: rows split R ways, columns C ways. Column vectors split C ways (duplicated
    across the column group), row vectors (tok2.b) split R ways (duplicated across the row
    group). With (R, C) = (1, 2) / (2, 2) this equals the reference Layout.local at n = 2 / 4
    (model.py:135-150): at n = 4 position pos = 2 r + c.
    """
    spec = {s[0]: s for s in param_specs(cfg)}[name]
    _, _, _, kind, row_ax, col_ax, _, _ = spec
    if kind == "matrix":
        rows = axis_sets(cfg, row_ax, R)[r] if R > 1 else slice(None)
        cols = axis_sets(cfg, col_ax, C)[c] if C > 1 else slice(None)
        return np.ascontiguousarray(glob[rows][:, cols])
    if kind == "vec_col":
        return np.ascontiguousarray(glob[axis_sets(cfg, col_ax, C)[c]] if C > 1 else glob)
    return np.ascontiguousarray(glob[axis_sets(cfg, row_ax, R)[r]] if R > 1 else glob)


def ref_layout_local(cfg: Config, name: str, glob: np.ndarray, n: int, pos: int) -> np.ndarray:
    """Reference Layout.local (model.py:135-150) for n in {1, 2, 4}."""
    if n == 1:
        return glob.copy()
    if n == 2:
        return local_tile(cfg, name, glob, 1, 2, 0, pos)
    return local_tile(cfg, name, glob, 2, 2, pos // 2, pos % 2)


def local_sample(cfg: Config, x: np.ndarray, R: int, C: int, r: int, c: int) -> np.ndarray:
    """[B, lat, lon, vars] -> rank (r, c)'s block: longitude part r, channel part c (SPEC 4.2)."""
    lon_sets = contiguous_split(cfg.grid[1], R) if R > 1 else [np.arange(cfg.grid[1])]
    ch_sets = contiguous_split(cfg.n_vars, C) if C > 1 else [np.arange(cfg.n_vars)]
    return np.ascontiguousarray(x[:, :, lon_sets[r]][..., ch_sets[c]])


# --------------------------------------------------------------------------- serial model
class SerialModel:
    """n = 1 WeatherMixer forward/backward (model.py:406-445) over global numpy params."""

    def __init__(self, cfg: Config, params: dict, eps: float = 1e-5):
        self.cfg, self.p, self.eps = cfg, params, eps
        self._cache = None

    def _ln(self, x, pre):
        s, sq = ops.row_moments(x)
        y, xhat, inv = ops.ln_from_moments(x, s, sq, x.shape[-1], self.p[pre + "gamma"], self.p[pre + "beta"], self.eps)
        return y, (xhat, inv)

    def block_forward(self, i: int, h):
        """MixerBlock.forward (model.py:268-282) at n = 1."""
        p, b = self.p, f"block{i}."
        u, c_ln1 = self._ln(h, b + "ln1.")
        t1 = ops.matmul(u, p[b + "tok1.w"], "TN") + p[b + "tok1.b"]          # [B, E, K]
        a = ops.gelu(t1)
        o = ops.matmul(p[b + "tok2.w"], a, "NT") + p[b + "tok2.b"][:, None]  # [B, T, E]
        x2 = h + o
        v, c_ln2 = self._ln(x2, b + "ln2.")
        cc = ops.matmul(v, p[b + "ch1.w"], "NT") + p[b + "ch1.b"]
        ca = ops.gelu(cc)
        z = ops.matmul(ca, p[b + "ch2.w"], "NT") + p[b + "ch2.b"]
        return x2 + z, (h, c_ln1, u, t1, a, c_ln2, v, cc, ca)

    def block_backward(self, i: int, cache, gh, grads):
        """MixerBlock.backward (model.py:284-297) at n = 1; accumulates into grads."""
        p, b, cfg = self.p, f"block{i}.", self.cfg
        h, c_ln1, u, t1, a, c_ln2, v, cc, ca = cache
        grads[b + "ch2.w"] += _flat(ops.matmul(gh, ca, "TN"))
        grads[b + "ch2.b"] += gh.sum(axis=(0, 1))
        g_c = ops.gelu_backward(cc, ops.matmul(gh, p[b + "ch2.w"], "NN"))
        grads[b + "ch1.w"] += _flat(ops.matmul(g_c, v, "TN"))
        grads[b + "ch1.b"] += g_c.sum(axis=(0, 1))
        g_v = ops.matmul(g_c, p[b + "ch1.w"], "NN")
        dx, dgam, dbet = ops.ln_backward_from_cache(g_v, p[b + "ln2.gamma"], *c_ln2, cfg.d_emb)
        grads[b + "ln2.gamma"] += dgam
        grads[b + "ln2.beta"] += dbet
        g_x2 = gh + dx
        # tok2 (weight-first NT): dW += sum_b g @ a ; ga = g^T W ; db(row) += sum g over E
        grads[b + "tok2.w"] += _flat(ops.matmul(g_x2, a, "NN"))
        grads[b + "tok2.b"] += g_x2.sum(axis=tuple(i2 for i2 in range(g_x2.ndim) if i2 != g_x2.ndim - 2))
        g_t1 = ops.gelu_backward(t1, ops.matmul(g_x2, p[b + "tok2.w"], "TN"))
        # tok1 (TN): gu = W g^T ; dW += sum_b u @ g ; db += sum over (B, E)
        grads[b + "tok1.w"] += _flat(ops.matmul(u, g_t1, "NN"))
        grads[b + "tok1.b"] += g_t1.sum(axis=(0, 1))
        g_u = ops.matmul(p[b + "tok1.w"], g_t1, "NT")
        dx, dgam, dbet = ops.ln_backward_from_cache(g_u, p[b + "ln1.gamma"], *c_ln1, cfg.d_emb)
        grads[b + "ln1.gamma"] += dgam
        grads[b + "ln1.beta"] += dbet
        return g_x2 + dx

    def forward(self, x, r: int = 1):
        cfg, p = self.cfg, self.p
        xp = ops.patchify(x, *cfg.patch)
        h = ops.matmul(xp, p["enc.w"], "NT") + p["enc.b"]
        enc_in = xp
        passes = []
        for _ in range(r):
            caches = []
            for i in range(cfg.n_blocks):
                h, cache = self.block_forward(i, h)
                caches.append(cache)
            passes.append(caches)
        d = ops.matmul(h, p["dec.w"], "NT") + p["dec.b"]
        decoded = ops.unpatchify(d, cfg.grid[0], cfg.grid[1], *cfg.patch)
        w = p["blend.w"]
        out = w * decoded + (1.0 - w) * x
        self._cache = (x, enc_in, passes, h, decoded)
        return out

    def backward(self, g_out):
        if self._cache is None:
            raise RuntimeError("backward called without a cached forward")
        x, xp, passes, hdec, decoded = self._cache
        self._cache = None
        cfg, p = self.cfg, self.p
        grads = {k: np.zeros_like(v) for k, v in p.items()}
        lead = tuple(range(g_out.ndim - 1))
        grads["blend.w"] += (g_out * (decoded - x)).sum(axis=lead)
        g = ops.patchify(g_out * p["blend.w"], *cfg.patch)
        # decoder (NT): gx = g W ; dW += sum_b g^T h ; db += sum g
        grads["dec.w"] += _flat(ops.matmul(g, hdec, "TN"))
        grads["dec.b"] += g.sum(axis=(0, 1))
        gh = ops.matmul(g, p["dec.w"], "NN")
        for caches in reversed(passes):
            for i in reversed(range(cfg.n_blocks)):
                gh = self.block_backward(i, caches[i], gh, grads)
        grads["enc.w"] += _flat(ops.matmul(gh, xp, "TN"))
        grads["enc.b"] += gh.sum(axis=(0, 1))
        return grads


def _flat(a):
    """parallel.py:552-556."""
    return a if a.ndim == 2 else a.sum(axis=tuple(range(a.ndim - 2)))


def train_flops(cfg: Config, batch: int = 1, r: int = 1) -> int:
    """3 * B * [4 T F E + r n_blocks 4 T E (d_tok + d_ch)] (= sum MpContext.flops)."""
    T, F, E = cfg.tokens, cfg.patch_features, cfg.d_emb
    return 3 * batch * (4 * T * F * E + r * cfg.n_blocks * 4 * T * E * (cfg.d_tok + cfg.d_ch))
