"""ORACLE — TEST INFRASTRUCTURE ONLY. Never imported by the product package.

A CPU (numpy/scipy) restatement of the reference `jigsaw` 0.1.0 algorithm for the
WeatherMixer training step (reference /root/reference/pkg/src/jigsaw), used as

  * the parity checker of the sm_100a path (tests/, __graft_entry__.smoke()), and
  * the `cpu_baseline` / `--impl reference` timing arm of bench.py (kind "port": the
    reference is pure Python, so there is nothing to compile into oracle/_ref; the GPU
    box has no /root/reference, so the port travels instead).

Only tests/, __graft_entry__.smoke() and bench.py's CPU-baseline leg may import it.

Pinning: the port is checked against
  - the reference's own known-answer tests for this path (test_tensor.py fixed vectors),
  - golden vectors produced by running the reference itself in the build container
    (tests/golden/make_golden.py -> tests/golden/*.npz): model init bit-exact, forward
    output and every parameter gradient at n=1 (and the n=2 / n=4 runs) to <= 1e-12,
    analytic communication volumes exactly.
Loss and Adam have no reference code; they are restated from
SPEC and pinned to SPEC's worked examples only ("parity pinned to SPEC examples").

Modules
  ops.py      tensor.py restatement (matmul modes, GELU, layer norm, patchify, dropout)
  model.py    ModelConfig / init / serial forward+backward (model.py, parallel.py at n=1),
              per-rank layouts (Layout.local, model.py:124-197), grid-R x C tile maps
  train.py    lat weights + lat-weighted MSE (SPEC data module), Adam (SPEC train module)
  volume.py   analytic communication volume (parallel.py:361-466, model.py:483-529)
"""
