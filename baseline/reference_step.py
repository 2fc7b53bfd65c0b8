"""The reference arm of bench.py: one WeatherMixer training step of the UNMODIFIED reference
package (`jigsaw` 0.1.0, pure numpy, installed into baseline/_ref by

    python -m pip install --no-index --no-build-isolation --find-links /opt/wheelhouse \
        --target baseline/_ref <copy of /root/reference/pkg> --no-deps

— see DESIGN.md §6), run through its own public API and stock code path on the host cores:

    model.zero_grads() -> model.forward(x) -> SPEC loss + dL/dout -> model.backward(g)
    -> model.grad_sync() -> Adam on every Param

(reference model.py:406-460). The reference ships no loss or optimiser; those two
steps use the SPEC restatement in oracle/train.py (SPEC.md:396-407 loss, 482-490 Adam), the
same conventions the B200 step implements. Nothing of the B200 package is on this path.

n = 1 (one rank, `InProcWorld(1)`): the reference's fastest configuration on one host — its
thread-SPMD ranks share the same cores and BLAS pool and run slower with n.
"""
from __future__ import annotations

import os
import sys
import time

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
REF = os.path.join(HERE, "_ref")


def load_reference():
    """Import the installed reference package (baseline/_ref/jigsaw); None when absent."""
    if not os.path.isdir(os.path.join(REF, "jigsaw")):
        return None
    if REF not in sys.path:
        sys.path.insert(0, REF)
    import jigsaw  # noqa: F401
    from jigsaw import comm as rcomm, model as rmodel, parallel as rpar
    return rcomm, rmodel, rpar


def host_cores() -> int:
    try:
        return len(os.sched_getaffinity(0))
    except AttributeError:  # pragma: no cover
        return os.cpu_count() or 1


def cpu_model() -> str:
    try:
        for ln in open("/proc/cpuinfo"):
            if ln.startswith("model name"):
                return ln.split(":", 1)[1].strip()
    except OSError:
        pass
    return "unknown"


class ReferenceStep:
    """A reference WeatherMixerModel (f32, n = 1) plus the SPEC loss and Adam state."""

    def __init__(self, cfg_kw: dict, lat_real: int, vars_real: int, batch: int = 1, seed: int = 0):
        mods = load_reference()
        if mods is None:
            raise RuntimeError(f"reference package not installed under {REF}")
        rcomm, rmodel, rpar = mods
        sys.path.insert(0, os.path.dirname(HERE))
        from oracle import train as ot
        self.ot = ot
        cfg = rmodel.ModelConfig(**{k: (tuple(v) if isinstance(v, list) else v) for k, v in cfg_kw.items()})
        comm = rcomm.InProcWorld(1).communicator(0)
        self.ctx = rpar.MpContext(comm, [0])
        t0 = time.perf_counter()
        self.model = rmodel.WeatherMixerModel(self.ctx, cfg, seed=seed, dtype="f32")
        self.init_s = time.perf_counter() - t0
        self.cfg, self.batch = cfg, batch
        lat, lon = cfg.grid
        rng = np.random.default_rng(1234)
        shape = (batch, lat, lon, cfg.n_vars)
        self.x = rng.standard_normal(shape, dtype=np.float32)
        self.target = rng.standard_normal(shape, dtype=np.float32)
        for a in (self.x, self.target):
            a[:, lat_real:] = 0
            a[..., vars_real:] = 0
        self.lat_w = ot.lat_weights(lat, lat_real).astype(np.float32)
        self.var_w = np.zeros(cfg.n_vars, np.float32)
        self.var_w[:vars_real] = 1.0
        self.count = batch * lat_real * lon * vars_real
        self.m = {k: np.zeros_like(p.data) for k, p in self.model.params.items()}
        self.v = {k: np.zeros_like(p.data) for k, p in self.model.params.items()}
        self.t = 0
        self.lr = {"body": 1e-4, "encdec": 2e-5}  # PAPER.md:305; lr classes model.py:336-338

    def step(self) -> float:
        m = self.model
        m.zero_grads()
        out = m.forward(self.x)
        loss, g = self.ot.weighted_mse_loss(out, self.target, self.lat_w, self.var_w, self.count)
        m.backward(g.astype(np.float32))
        m.grad_sync()
        self.t += 1
        for k, p in m.params.items():
            self.ot.adam_step(p.data, p.grad, self.m[k], self.v[k], self.t, self.lr[p.lr_class])
        return loss

    def flops(self) -> int:
        return self.ctx.flops


def blas_threads(n: int):
    """Context that runs numpy's BLAS on n threads. torchrun exports OMP_NUM_THREADS=1 to every
    rank, which OpenBLAS reads at load time; the reference arm (rank 0 alone) should use all the
    host threads whatever the launcher, so the pool is resized at run time (threadpoolctl)."""
    try:
        from threadpoolctl import threadpool_limits
        return threadpool_limits(limits=n, user_api="blas")
    except Exception:  # noqa: BLE001
        import contextlib
        return contextlib.nullcontext()


def blas_thread_count() -> int | None:
    try:
        from threadpoolctl import threadpool_info
        return max((i.get("num_threads") or 0) for i in threadpool_info() if i.get("user_api") == "blas") or None
    except Exception:  # noqa: BLE001
        return None


def time_steps(cfg_kw, lat_real, vars_real, batch, warmup, steps, budget_s):
    """(per-step seconds list, warm-ups actually run, init seconds, loss) — warm-up and timed
    steps are capped so the whole run stays inside budget_s (estimated from the first step).
    BLAS runs on every host thread (see blas_threads)."""
    with blas_threads(host_cores()):
        return _time_steps(cfg_kw, lat_real, vars_real, batch, warmup, steps, budget_s)


def _time_steps(cfg_kw, lat_real, vars_real, batch, warmup, steps, budget_s):
    rs = ReferenceStep(cfg_kw, lat_real, vars_real, batch)
    rs.blas_threads = blas_thread_count()  # the pool size the timed steps actually ran with
    times, warm_done, loss = [], 0, float("nan")
    t_first = None
    for _ in range(max(0, warmup)):
        t0 = time.perf_counter()
        loss = rs.step()
        t_first = time.perf_counter() - t0
        warm_done += 1
        if t_first * (warm_done + 1) > 0.4 * budget_s:
            break
    while len(times) < max(1, steps):
        t0 = time.perf_counter()
        loss = rs.step()
        times.append(time.perf_counter() - t0)
        spent = sum(times) + (t_first or 0) * warm_done
        if spent + times[-1] > budget_s:
            break
    return times, warm_done, rs.init_s, loss, rs
