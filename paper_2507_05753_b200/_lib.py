"""ctypes binding of libjigsaw_sm100.so (the C ABI declared in include/jigsaw_sm100.h).

This is the only place the package touches the native library. Every wrapper takes torch
CUDA tensors (torch is used for device memory and streams only), passes raw pointers and
the current stream, and maps the library's status codes onto the reference's exceptions:
JG_ERR_SHAPE -> ShapeError (reference tensor.py:23), JG_ERR_CUDA -> RuntimeError.

There is no fallback: if the library is missing or cannot be loaded the import of any
compute entry point raises.
"""
from __future__ import annotations

import ctypes
import os
from pathlib import Path

import torch

from .errors import ShapeError

_PKG = Path(__file__).resolve().parent
LIB_PATH = _PKG / "libjigsaw_sm100.so"

JG_OK, JG_ERR_SHAPE, JG_ERR_CUDA = 0, 1, 2
JG_F32, JG_BF16 = 0, 1
JG_KMAJOR, JG_MNMAJOR = 0, 1
JG_MATH_BF16, JG_MATH_TF32X3 = 0, 1
EPI_ACCUM, EPI_BIAS_COL, EPI_BIAS_ROW, EPI_RESID = 1, 2, 4, 8
EPI_GELU_FWD, EPI_GELU_BWD, EPI_COPY_D2, EPI_STATS = 16, 32, 64, 128
EPI_ADAM = 256
EPI_LNB = 512

EXPORTED = [
    "jg_gemm", "jg_split_tf32", "jg_split_tf32_2d", "jg_cast_bf16", "jg_gelu_fwd", "jg_gelu_bwd",
    "jg_ln_moments", "jg_ln_apply", "jg_ln_bwd_moments", "jg_ln_bwd_apply",
    "jg_colsum", "jg_rowsum", "jg_patchify", "jg_unpatchify", "jg_blend_loss",
    "jg_adam", "jg_adam_sms", "jg_adam_push", "jg_step_increment", "jg_sqnorm", "jg_epilogue", "jg_axpy", "jg_sum_planes", "jg_copy_async", "jg_push", "jg_memset",
    "jg_group_barrier", "jg_opt_schedule", "jg_version", "jg_last_error", "jg_launch_count",
    "jg_gemm_desc_size",
]
JG_MAX_LR_CLASSES = 4


class Bcast(ctypes.Structure):
    """jg_bcast: up to 4 extra destinations of an output (peer gather slots)."""
    _fields_ = [("ptr", ctypes.c_void_p * 4), ("n", ctypes.c_int32)]


_NUM_SMS = None


def num_sms() -> int:
    """SM count of the current device (148 on B200)."""
    global _NUM_SMS
    if _NUM_SMS is None:
        import torch
        _NUM_SMS = torch.cuda.get_device_properties(torch.cuda.current_device()).multi_processor_count
    return _NUM_SMS


def make_bcast(addrs) -> "Bcast | None":
    if not addrs:
        return None
    if len(addrs) > 4:
        raise ValueError("at most 4 broadcast destinations")
    b = Bcast()
    for i, a in enumerate(addrs):
        b.ptr[i] = a
    b.n = len(addrs)
    return b


JG_MAX_PUSH_SEGS = 16


class PushSeg(ctypes.Structure):
    """jg_push_seg: a range of an Adam call whose bf16 copy is also stored at up to 4 addresses."""
    _fields_ = [("start", ctypes.c_int64), ("len", ctypes.c_int64), ("dst", ctypes.c_void_p * 4),
                ("ndst", ctypes.c_int32)]


class PushTable(ctypes.Structure):
    _fields_ = [("seg", PushSeg * JG_MAX_PUSH_SEGS), ("nseg", ctypes.c_int32)]


def make_push_table(segs) -> "PushTable | None":
    """segs: [(start, len, [addr, ...]), ...] relative to the Adam call's range."""
    if not segs:
        return None
    if len(segs) > JG_MAX_PUSH_SEGS:
        raise ValueError(f"at most {JG_MAX_PUSH_SEGS} push segments")
    t = PushTable()
    for k, (start, n, addrs) in enumerate(segs):
        if len(addrs) > 4:
            raise ValueError("at most 4 push destinations")
        t.seg[k].start, t.seg[k].len, t.seg[k].ndst = start, n, len(addrs)
        for d, a in enumerate(addrs):
            t.seg[k].dst[d] = a
    t.nseg = len(segs)
    return t


class LrSchedule(ctypes.Structure):
    """jg_lr_schedule."""
    _fields_ = [("base_lr", ctypes.c_float), ("warm_start", ctypes.c_float), ("final_lr", ctypes.c_float),
                ("warmup_steps", ctypes.c_int64), ("total_steps", ctypes.c_int64)]


class GemmDesc(ctypes.Structure):
    _fields_ = [
        ("m", ctypes.c_int64), ("n", ctypes.c_int64), ("k", ctypes.c_int64), ("batch", ctypes.c_int64),
        ("math", ctypes.c_int32), ("reduce_batch", ctypes.c_int32),
        ("a", ctypes.c_void_p), ("a_lo", ctypes.c_void_p), ("lda", ctypes.c_int64), ("a_bstride", ctypes.c_int64),
        ("a_major", ctypes.c_int32),
        ("b", ctypes.c_void_p), ("b_lo", ctypes.c_void_p), ("ldb", ctypes.c_int64), ("b_bstride", ctypes.c_int64),
        ("b_major", ctypes.c_int32),
        ("epi", ctypes.c_uint32), ("alpha", ctypes.c_float),
        ("d", ctypes.c_void_p), ("ldd", ctypes.c_int64), ("d_bstride", ctypes.c_int64), ("d_type", ctypes.c_int32),
        ("d2", ctypes.c_void_p), ("ldd2", ctypes.c_int64), ("d2_bstride", ctypes.c_int64), ("d2_type", ctypes.c_int32),
        ("bias", ctypes.c_void_p), ("bias_bstride", ctypes.c_int64),
        ("resid", ctypes.c_void_p), ("ldr", ctypes.c_int64), ("r_bstride", ctypes.c_int64),
        ("pre", ctypes.c_void_p), ("ldp", ctypes.c_int64), ("p_bstride", ctypes.c_int64), ("pre_type", ctypes.c_int32),
        ("stats", ctypes.c_void_p), ("stats_bstride", ctypes.c_int64),
        ("adam_m", ctypes.c_void_p), ("adam_v", ctypes.c_void_p), ("adam_pbf16", ctypes.c_void_p),
        ("adam_step", ctypes.c_void_p), ("adam_lr", ctypes.c_float), ("adam_beta1", ctypes.c_float),
        ("adam_beta2", ctypes.c_float), ("adam_eps", ctypes.c_float),
        ("d_planes", ctypes.c_void_p * 8),
        ("d_bcast", Bcast), ("d2_bcast", Bcast),
        ("rs_flags", ctypes.c_void_p), ("rs_flag_peers", ctypes.c_void_p * 8),
        ("rs_src", ctypes.c_void_p), ("rs_src_stride", ctypes.c_int64),
        ("rs_part_type", ctypes.c_int32), ("rs_nsrc", ctypes.c_int32), ("rs_src_idx", ctypes.c_int32),
        ("rs_own", ctypes.c_int32), ("rs_need", ctypes.c_int32), ("rs_flag_cap", ctypes.c_int32),
        ("lnb_x", ctypes.c_void_p), ("lnb_ldx", ctypes.c_int64), ("lnb_x_bstride", ctypes.c_int64),
        ("lnb_gamma", ctypes.c_void_p), ("lnb_mr", ctypes.c_void_p),
        ("max_sms", ctypes.c_int32),
        ("plane_div", ctypes.c_int32), ("d_planes_bstride", ctypes.c_int64),
        ("tile_n", ctypes.c_int32),
    ]


_lib = None


def load(path: str | os.PathLike | None = None) -> ctypes.CDLL:
    """Load (once) and return the native library; raises if it is absent."""
    global _lib
    if _lib is not None:
        return _lib
    # JIGSAW_LIB: load another build of the same library (A/B timing of kernel changes, tools/ab.sh)
    p = Path(path) if path else Path(os.environ.get("JIGSAW_LIB", LIB_PATH))
    if not p.exists():
        raise RuntimeError(
            f"{p} not found: build it with `python -c 'import __graft_entry__ as g; g.build()'` "
            "(no CPU fallback exists by design)")
    lib = ctypes.CDLL(str(p))
    vp, i64, i32, f32 = ctypes.c_void_p, ctypes.c_int64, ctypes.c_int32, ctypes.c_float
    sig = {
        "jg_gemm": [ctypes.POINTER(GemmDesc), vp],
        "jg_split_tf32": [vp, vp, vp, i64, vp],
        "jg_split_tf32_2d": [vp, i64, i64, i64, i64, i64, i32, vp, vp, i64, vp],
        "jg_cast_bf16": [vp, vp, i64, vp],
        "jg_gelu_fwd": [vp, vp, i32, i64, vp],
        "jg_gelu_bwd": [vp, vp, vp, i32, i64, vp],
        "jg_ln_moments": [vp, vp, i64, i64, i64, vp],
        "jg_ln_apply": [vp, vp, vp, vp, vp, i32, vp, i64, i64, i64, f32, vp, vp],
        "jg_ln_bwd_moments": [vp, vp, vp, vp, vp, i64, i64, vp],
        "jg_ln_bwd_apply": [vp, vp, vp, vp, vp, vp, vp, vp, vp, vp, vp, i64, vp, i64, i64, i64, vp, vp],
        "jg_colsum": [vp, i32, vp, i64, i64, i64, vp],
        "jg_rowsum": [vp, i32, vp, i64, i64, i64, vp],
        "jg_patchify": [vp, vp, i32, i64, i64, i64, i64, i64, i64, vp],
        "jg_unpatchify": [vp, vp, i64, i64, i64, i64, i64, i64, vp],
        "jg_blend_loss": [vp] * 12 + [i64] * 6 + [f32, f32, vp, vp],
        "jg_adam": [vp, vp, vp, vp, vp, i64, f32, f32, f32, f32, vp, vp, vp, vp],
        "jg_adam_sms": [vp, vp, vp, vp, vp, i64, f32, f32, f32, f32, vp, vp, vp, i32, vp],
        "jg_adam_push": [vp, vp, vp, vp, vp, i64, f32, f32, f32, f32, vp, vp, vp, ctypes.POINTER(PushTable), vp],
        "jg_step_increment": [vp, vp],
        "jg_sqnorm": [vp, i64, f32, vp, vp],
        "jg_opt_schedule": [vp, ctypes.POINTER(LrSchedule), i32, vp, f32, vp, vp, vp],
        "jg_epilogue": [ctypes.POINTER(GemmDesc), vp, i32, i64, i64, i32, vp],
        "jg_axpy": [vp, vp, f32, i64, vp],
        "jg_sum_planes": [vp, vp, i32, i64, i32, i64, i32, vp],
        "jg_copy_async": [vp, vp, i64, vp],
        "jg_push": [vp, i64, vp, vp],
        "jg_memset": [vp, i64, vp],
        "jg_group_barrier": [ctypes.POINTER(ctypes.c_void_p), vp, vp, i32, i32, vp],
    }
    for name, args in sig.items():
        fn = getattr(lib, name)
        fn.argtypes = args
        fn.restype = ctypes.c_int
    lib.jg_version.restype = ctypes.c_char_p
    lib.jg_last_error.restype = ctypes.c_char_p
    lib.jg_launch_count.restype = ctypes.c_int64
    lib.jg_gemm_desc_size.restype = ctypes.c_size_t
    if lib.jg_gemm_desc_size() != ctypes.sizeof(GemmDesc):
        raise RuntimeError(f"{path}: jg_gemm_desc is {lib.jg_gemm_desc_size()} bytes in the library, "
                           f"{ctypes.sizeof(GemmDesc)} in _lib.GemmDesc (stale build?)")
    _lib = lib
    return lib


def version() -> str:
    return load().jg_version().decode()


def launch_count() -> int:
    return int(load().jg_launch_count())


def _check(rc: int, what: str) -> None:
    if rc == JG_OK:
        return
    msg = load().jg_last_error().decode()
    if rc == JG_ERR_SHAPE:
        raise ShapeError(f"{what}: {msg}")
    raise RuntimeError(f"{what}: {msg}")


def call(name: str, *args) -> None:
    """Invoke one C entry point; the trailing stream argument is appended here."""
    lib = load()
    stream = torch.cuda.current_stream().cuda_stream
    _check(getattr(lib, name)(*args, ctypes.c_void_p(stream)), name)


def ptr(t: torch.Tensor | None) -> int | None:
    return None if t is None else t.data_ptr()


def dtype_code(t: torch.Tensor) -> int:
    if t.dtype == torch.float32:
        return JG_F32
    if t.dtype == torch.bfloat16:
        return JG_BF16
    raise ShapeError(f"unsupported dtype {t.dtype}")


def gemm_raw(desc: GemmDesc) -> None:
    lib = load()
    stream = torch.cuda.current_stream().cuda_stream
    _check(lib.jg_gemm(ctypes.byref(desc), ctypes.c_void_p(stream)), "jg_gemm")
