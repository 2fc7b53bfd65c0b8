"""ORACLE (test infrastructure): numpy restatement of reference tensor.py.

Each function cites the reference line range it follows. f32/f64 numpy arrays.
"""
from __future__ import annotations

import numpy as np
from scipy.special import erf

_SQRT_HALF = 0.7071067811865476
_INV_SQRT_2PI = 0.3989422804014327


class OracleShapeError(ValueError):
    pass


def matmul(a: np.ndarray, b: np.ndarray, mode: str = "NN") -> np.ndarray:
    """NN a@b, NT a@b^T, TN a^T@b with broadcast batch dims (tensor.py:43-72)."""
    if a.dtype != b.dtype:
        raise OracleShapeError(f"matmul dtype mismatch: {a.dtype} vs {b.dtype}")
    if a.ndim < 2 or b.ndim < 2:
        raise OracleShapeError(f"matmul needs >=2-D operands, got {a.shape} and {b.shape}")
    mode = str(getattr(mode, "value", mode))
    if mode == "NN":
        if a.shape[-1] != b.shape[-2]:
            raise OracleShapeError(f"matmul NN: incompatible shapes {a.shape} and {b.shape}")
        return np.matmul(a, b)
    if mode == "NT":
        if a.shape[-1] != b.shape[-1]:
            raise OracleShapeError(f"matmul NT: incompatible shapes {a.shape} and {b.shape}")
        return np.matmul(a, np.swapaxes(b, -1, -2))
    if a.shape[-2] != b.shape[-2]:
        raise OracleShapeError(f"matmul TN: incompatible shapes {a.shape} and {b.shape}")
    return np.matmul(np.swapaxes(a, -1, -2), b)


def gelu(x):
    """x * Phi(x), exact erf (tensor.py:75-77)."""
    return x * (0.5 * (1.0 + erf(x * _SQRT_HALF)))


def gelu_backward(x, upstream):
    """upstream * (Phi(x) + x phi(x)) (tensor.py:80-84)."""
    pdf = np.exp(-0.5 * x * x) * _INV_SQRT_2PI
    cdf = 0.5 * (1.0 + erf(x * _SQRT_HALF))
    return upstream * (cdf + x * pdf)


def row_moments(x):
    """(sum x, sum x^2) over the last axis — the one-pass formula of tensor.py:87-94."""
    return x.sum(axis=-1), (x * x).sum(axis=-1)


def ln_from_moments(x, s, sq, c_total, gamma, beta, eps):
    """Normalise with given row totals (model.py:233-240); returns y, xhat, inv_std."""
    mean = s[..., None] / c_total
    var = sq[..., None] / c_total - mean * mean
    inv_std = 1.0 / np.sqrt(var + eps)
    xhat = (x - mean) * inv_std
    return gamma * xhat + beta, xhat, inv_std


def layer_norm(x, gamma, beta, eps=1e-5):
    """tensor.py:97-106."""
    if eps <= 0:
        raise ValueError(f"layer_norm eps must be > 0, got {eps}")
    s, sq = row_moments(x)
    y, _, _ = ln_from_moments(x, s, sq, x.shape[-1], gamma, beta, eps)
    return y


def ln_backward_from_cache(g, gamma, xhat, inv_std, c_total, sh=None, shx=None):
    """model.py:242-250 (row sums may be supplied already reduced across ranks)."""
    h = g * gamma
    if sh is None:
        sh, shx = h.sum(axis=-1), (h * xhat).sum(axis=-1)
    dx = inv_std * (h - sh[..., None] / c_total - xhat * shx[..., None] / c_total)
    axes = tuple(range(g.ndim - 1))
    return dx, (g * xhat).sum(axis=axes), g.sum(axis=axes)


def layer_norm_backward(x, gamma, eps, upstream):
    """tensor.py:109-123."""
    if eps <= 0:
        raise ValueError(f"layer_norm eps must be > 0, got {eps}")
    c = x.shape[-1]
    s, sq = row_moments(x)
    _, xhat, inv_std = ln_from_moments(x, s, sq, c, np.ones_like(x[..., :1]), 0.0, eps)
    return ln_backward_from_cache(upstream, gamma, xhat, inv_std, c)


def patchify(x, p_lat, p_lon):
    """[B, lat, lon, C] -> [B, tokens, C*p_lat*p_lon] (tensor.py:126-139)."""
    b, lat, lon, c = x.shape
    if lat % p_lat or lon % p_lon:
        raise OracleShapeError(f"grid {lat}x{lon} not divisible by patch {p_lat}x{p_lon}")
    gl, gw = lat // p_lat, lon // p_lon
    t = x.reshape(b, gl, p_lat, gw, p_lon, c).transpose(0, 1, 3, 5, 2, 4)
    return np.ascontiguousarray(t.reshape(b, gl * gw, c * p_lat * p_lon))


def unpatchify(tokens, lat, lon, p_lat, p_lon):
    """Inverse of patchify (tensor.py:142-151)."""
    b, n_tok, feat = tokens.shape
    gl, gw = lat // p_lat, lon // p_lon
    if n_tok != gl * gw or feat % (p_lat * p_lon):
        raise OracleShapeError(f"token tensor {tokens.shape} does not fit grid {lat}x{lon}")
    c = feat // (p_lat * p_lon)
    t = tokens.reshape(b, gl, gw, c, p_lat, p_lon).transpose(0, 1, 4, 2, 5, 3)
    return np.ascontiguousarray(t.reshape(b, lat, lon, c))


def dropout_mask(shape, rate, rng):
    """tensor.py:154-160."""
    if not 0.0 <= rate < 1.0:
        raise ValueError(f"dropout rate must be in [0, 1), got {rate}")
    if rate == 0.0:
        return None
    return (rng.random(shape) >= rate) / (1.0 - rate)
