"""Exception types of the reference `jigsaw` package, same names and bases.

ShapeError  — tensor.py:23        (ValueError)
ConfigError — model.py:37         (ValueError)
CommError   — comm.py:41          (RuntimeError); CommTimeout — comm.py:45
WorkerError — runtime.py:13       (RuntimeError, carries the failing rank)
"""


class ShapeError(ValueError):
    """Operand shapes incompatible with the requested operation."""


class ConfigError(ValueError):
    """Invalid experiment or model configuration; message names the field."""


class CommError(RuntimeError):
    """Transport-level failure (bad peer, duplicate tag, shutdown, ...)."""


class CommTimeout(CommError):
    """Deadlock guard: a wait exceeded its timeout."""


class WorkerError(RuntimeError):
    def __init__(self, rank: int, tb: str):
        super().__init__(f"rank {rank} failed:\n{tb}")
        self.rank = rank
        self.tb = tb
