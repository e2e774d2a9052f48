"""ctypes binding of ``libtreepipe_b200.so`` (the C ABI in include/treepipe_b200.h).

There is no CPU fallback: if the library is missing or no CUDA device is
visible, :func:`lib` raises.  ctypes releases the GIL for every call, so
distinct stages can be driven from worker threads (reference worker mode,
`pipeline.py:195-199`).
"""

from __future__ import annotations

import ctypes as C
import os
import threading

from .errors import ConfigError, ContractViolation, InvariantViolation, ShapeError

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "libtreepipe_b200.so")
if os.environ.get("TP_LIB_VARIANT"):  # A/B experiments: an in-tree build variant, libtreepipe_b200.<name>.so
    LIB_PATH = os.path.join(HERE, f"libtreepipe_b200.{os.environ['TP_LIB_VARIANT']}.so")

TP_OK, TP_ESHAPE, TP_ECONTRACT, TP_EINVARIANT, TP_ECONFIG, TP_ECUDA = range(6)
ARCH_TOY, ARCH_LLAMA = 0, 1

_ERRORS = {
    TP_ESHAPE: ShapeError,
    TP_ECONTRACT: ContractViolation,
    TP_EINVARIANT: InvariantViolation,
    TP_ECONFIG: ConfigError,
    TP_ECUDA: InvariantViolation,
}


class ModelConfig(C.Structure):
    _fields_ = [
        ("arch", C.c_int32), ("vocab", C.c_int32), ("hidden", C.c_int32), ("layers", C.c_int32),
        ("heads", C.c_int32), ("kv_heads", C.c_int32), ("head_dim", C.c_int32), ("ffn", C.c_int32),
        ("layer_lo", C.c_int32), ("layer_hi", C.c_int32), ("with_embed", C.c_int32),
        ("with_head", C.c_int32), ("device", C.c_int32), ("max_nodes", C.c_int32),
        ("rope_theta", C.c_float), ("norm_eps", C.c_float), ("weight_scale", C.c_int32),
    ]


class Level(C.Structure):
    _fields_ = [
        ("n", C.c_int32), ("append", C.c_int32), ("tokens", C.c_void_p), ("positions", C.c_void_p),
        ("prefix_rows", C.c_void_p), ("words", C.c_int32), ("bits_base", C.c_int32),
        ("anc_bits", C.c_void_p), ("layer_lo", C.c_int32), ("layer_hi", C.c_int32),
        ("tree_bits", C.c_void_p), ("tree_lo", C.c_int32), ("tree_off", C.c_int32), ("tree_prefix", C.c_int32),
    ]


class Item(C.Structure):
    _fields_ = [("stage", C.c_void_p), ("level", Level), ("hidden_in", C.c_void_p), ("member", C.c_int32)]


class PruneStage(C.Structure):
    _fields_ = [("stage", C.c_void_p), ("prefix_rows", C.c_int32), ("spec_rows", C.c_int32),
                ("tree_off", C.c_int32), ("level_lo", C.c_int32), ("level_n", C.c_int32),
                ("hidden_src", C.c_void_p), ("hidden_dst", C.c_void_p), ("keep_out", C.c_void_p)]


_P = C.c_void_p
_I = C.c_int32
_SIGS = {
    "tp_prune_device": (C.c_int, [_I, _P, _P, _P, _I, _I, _P, _I, C.c_int64, _P]),
    "tp_result_mirror": (C.c_int, [_P, _P, _P]),
    "tp_peer_copy": (C.c_int, [_P, _I, _P, _I, C.c_int64, _P]),
    "tp_last_error": (C.c_char_p, []),
    "tp_device_count": (C.c_int, [C.POINTER(C.c_int32)]),
    "tp_model_create": (C.c_int, [C.POINTER(ModelConfig), C.POINTER(_P)]),
    "tp_model_destroy": (C.c_int, [_P]),
    "tp_model_init_lcg": (C.c_int, [_P, C.c_uint64, _P]),
    "tp_lcg_uniform": (C.c_int, [_I, C.c_uint64, C.c_int64, C.c_int64, _P, _P]),
    "tp_model_tensor_bytes": (C.c_int, [_P, _I, _I, C.POINTER(C.c_int64)]),
    "tp_model_write_tensor": (C.c_int, [_P, _I, _I, _P, C.c_int64]),
    "tp_model_read_tensor": (C.c_int, [_P, _I, _I, _P, C.c_int64]),
    "tp_model_embed": (C.c_int, [_P, _I, _P, _P, _P, _P]),
    "tp_model_logits": (C.c_int, [_P, _P, _I, _P, _P, _P]),
    "tp_model_verify": (C.c_int, [_P, _P, _P, _P, _I, _P, _P]),
    "tp_model_verify_async": (C.c_int, [_P, _P, _P, _P, _I, _P]),
    "tp_model_verify_wait": (C.c_int, [_P, _P]),
    "tp_stage_create": (C.c_int, [_P, _I, _I, _I, C.POINTER(_P)]),
    "tp_stage_destroy": (C.c_int, [_P]),
    "tp_stage_rows": (C.c_int, [_P, C.POINTER(C.c_int32)]),
    "tp_stage_reserve": (C.c_int, [_P, _I]),
    "tp_stage_forward": (C.c_int, [_P, C.POINTER(Level), _P, _P, _P]),
    "tp_stages_forward": (C.c_int, [_I, _P, _P, _P, _P, _P]),
    "tp_items_forward": (C.c_int, [_I, _P, _P, _P]),
    "tp_items_forward_ws": (C.c_int, [_I, _P, _P, _I, _P]),
    "tp_model_greedy_rows_async": (C.c_int, [_P, _P, _I, _P, _P]),
    "tp_model_greedy_rows_wait": (C.c_int, [_P, _I, _P]),
    "tp_stage_compact": (C.c_int, [_P, _I, _I, _P, _P]),
    "tp_stage_truncate": (C.c_int, [_P, _I]),
    "tp_stages_compact": (C.c_int, [_I, _P, _P, _P, _P, _P]),
    "tp_rows_compact_many": (C.c_int, [_I, _P, _P, _P, C.c_int64, _P, _P, _P, _P]),
    "tp_stage_read_kv": (C.c_int, [_P, _I, _I, _I, _I, _P]),
    "tp_rows_compact": (C.c_int, [_P, _P, _P, C.c_int64, _I, _P, C.POINTER(C.c_int32), _P]),
    "tp_debug_gemm": (C.c_int, [_I, _P, _P, _I, _I, _I, _P, _P]),
    "tp_debug_gemm_timed": (C.c_int, [_I, _P, _P, _I, _I, _I, _P, _I, _P, _P]),
    "tp_debug_gemm_group_timed": (C.c_int, [_I, _I, _P, _P, _P, _I, _I, _P, _I, _P, _P]),
    "tp_debug_argmax": (C.c_int, [_I, _P, _I, _I, _I, _P, _I, _P]),
    "tp_topk_rows": (C.c_int, [_I, _P, _I, _I, _I, _P, _P]),
    "tp_debug_gemm_hetero": (C.c_int, [_I, _I, _P, _P, _P, _P, _P, _P, _P]),
    "tp_debug_gemm_trace": (C.c_int, [_I, _P]),
    "tp_graph_launches": (C.c_int, [_P]),
    "tp_debug_gemm_knob": (C.c_int, [_I, _I]),
    "tp_synthetic_draft": (C.c_int, [C.c_uint64, C.c_int64, _I, C.c_double, C.c_double, C.c_double, _I, _I,
                                      _P, _P]),
    "tp_synthetic_draft_batch": (C.c_int, [_I, C.c_uint64, C.c_int64, _P, C.c_double, C.c_double, C.c_double,
                                            _I, _I, _P, _P]),
    "tp_debug_attn_tile": (C.c_int, [_I]),
    "tp_debug_attn_knob": (C.c_int, [_I, _I]),
    "tp_debug_attn_trace": (C.c_int, [C.c_void_p]),
    "tp_debug_dump": (C.c_int, [_P]),
    "tp_timeline_enable": (C.c_int, [_I]),
    "tp_timeline_read": (C.c_int, [C.c_char_p, _I]),
    "tp_launch_count": (C.c_int, [C.POINTER(C.c_int64)]),
    "tp_io_bytes": (C.c_int, [C.POINTER(C.c_int64), C.POINTER(C.c_int64)]),
    "tp_profile_enable": (C.c_int, [_I]),
    "tp_profile_read_members": (C.c_int, [_P, _P, _P]),
    "tp_profile_read": (C.c_int, [C.POINTER(C.c_double), C.POINTER(C.c_double), C.POINTER(C.c_int64)]),
}


def launch_count() -> int:
    n = C.c_int64()
    check(load().tp_launch_count(C.byref(n)))
    return n.value


def io_bytes() -> tuple[int, int]:
    h, d = C.c_int64(), C.c_int64()
    check(load().tp_io_bytes(C.byref(h), C.byref(d)))
    return h.value, d.value


_PROFILE_ON = False


def profile_enable(on: bool) -> None:
    global _PROFILE_ON
    _PROFILE_ON = bool(on)
    check(load().tp_profile_enable(int(on)))


class profile_paused:
    """Exclude a block's GEMM launches from the K2 roofline profile (the draft model's)."""

    def __enter__(self):
        self._was = _PROFILE_ON
        if self._was:
            check(load().tp_profile_enable(0))

    def __exit__(self, *a):
        if self._was:
            check(load().tp_profile_enable(1))
        return False


def profile_read_members() -> list[tuple[float, float, int]]:
    """(ms, bytes, launches) of the profiled GEMM launches, by member count 1..8."""
    ms, by, n = (C.c_double * 8)(), (C.c_double * 8)(), (C.c_int64 * 8)()
    check(load().tp_profile_read_members(ms, by, n))
    return [(ms[i], by[i], n[i]) for i in range(8)]


def profile_read() -> tuple[float, float, int]:
    ms, by, n = C.c_double(), C.c_double(), C.c_int64()
    check(load().tp_profile_read(C.byref(ms), C.byref(by), C.byref(n)))
    return ms.value, by.value, n.value

def timeline_enable(on: bool) -> None:
    check(load().tp_timeline_enable(int(on)))


def timeline_read() -> dict[str, float]:
    buf = C.create_string_buffer(1 << 16)
    check(load().tp_timeline_read(buf, len(buf)))
    out = {}
    for part in buf.value.decode().split(";"):
        if part:
            k, v = part.split("=")
            out[k] = float(v)
    return out


EXPORTED = tuple(_SIGS)

_lock = threading.Lock()
_lib: C.CDLL | None = None


def load(path: str = LIB_PATH) -> C.CDLL:
    """Load the shared library and declare every signature (no device needed)."""
    global _lib
    with _lock:
        if _lib is None:
            if not os.path.exists(path):
                raise InvariantViolation(
                    f"{path} missing: build it with `python -m paper_2504_04104_b200.build` "
                    "(there is no CPU fallback)")
            cdll = C.CDLL(path)
            for name, (res, args) in _SIGS.items():
                fn = getattr(cdll, name)
                fn.restype = res
                fn.argtypes = args
            _lib = cdll
    return _lib


def lib() -> C.CDLL:
    """The library, after checking a CUDA device is present."""
    import torch

    if not torch.cuda.is_available():
        raise InvariantViolation("no CUDA device visible: the B200 path has no CPU fallback")
    return load()


def check(status: int) -> None:
    if status == TP_OK:
        return
    msg = (load().tp_last_error() or b"").decode(errors="replace")
    raise _ERRORS.get(status, InvariantViolation)(msg or f"treepipe_b200 status {status}")


def ptr(arr) -> int | None:
    """Address of a numpy array / torch tensor (None for None)."""
    if arr is None:
        return None
    if hasattr(arr, "data_ptr"):
        return arr.data_ptr()
    return arr.ctypes.data


def stream_handle(stream=None) -> int:
    import torch

    s = stream if stream is not None else torch.cuda.current_stream()
    return s.cuda_stream
