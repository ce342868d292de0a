"""ctypes binding of libkvmix_b200.so (the C ABI in include/kvmix_b200.h).

This is the binding a Python caller of the reference would add. The
library is REQUIRED: there is no CPU fallback. Importing this module on a machine without
the built library raises immediately; calling a compute entry point without a CUDA device
returns KVMIX_CUDA_ERROR from the library, surfaced as KvmixCudaError.
"""
from __future__ import annotations

import ctypes as C
import os

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("KVMIX_LIB") or os.path.join(HERE, "libkvmix_b200.so")

OK, INVALID_ARGUMENT, OUT_OF_RANGE, RUNTIME_ERROR, CUDA_ERROR, OUT_OF_MEMORY = range(6)
F32, F16 = 0, 1
PER_CHANNEL_KEY, PER_TOKEN_VALUE = 0, 1


class KvmixError(Exception):
    status = RUNTIME_ERROR


class KvmixInvalidArgument(KvmixError, ValueError):
    """std::invalid_argument in the reference."""
    status = INVALID_ARGUMENT


class KvmixOutOfRange(KvmixError, IndexError):
    """std::out_of_range in the reference (PackedBuffer::get)."""
    status = OUT_OF_RANGE


class KvmixRuntimeError(KvmixError, RuntimeError):
    """std::runtime_error in the reference (deserialize / config parse / load)."""
    status = RUNTIME_ERROR


class KvmixCudaError(KvmixError, RuntimeError):
    status = CUDA_ERROR


class KvmixOutOfMemory(KvmixError, MemoryError):
    status = OUT_OF_MEMORY


_ERRORS = {
    INVALID_ARGUMENT: KvmixInvalidArgument,
    OUT_OF_RANGE: KvmixOutOfRange,
    RUNTIME_ERROR: KvmixRuntimeError,
    CUDA_ERROR: KvmixCudaError,
    OUT_OF_MEMORY: KvmixOutOfMemory,
}


class LayerConfigC(C.Structure):
    _fields_ = [("layer_index", C.c_int), ("key_bits", C.c_int), ("value_bits", C.c_int),
                ("key_rpc_ratio", C.c_float), ("value_rpc_ratio", C.c_float), ("group_size", C.c_int)]


class MemoryReportC(C.Structure):
    _fields_ = [("packed_payload_bits", C.c_uint64), ("metadata_bits", C.c_uint64), ("tail_bits", C.c_uint64),
                ("total_bits", C.c_uint64), ("fp16_baseline_bits", C.c_uint64), ("compression_ratio", C.c_double)]


_lib = None


def _declare(L):
    vp, i, i64, sz, u64 = C.c_void_p, C.c_int, C.c_int64, C.c_size_t, C.c_uint64
    sigs = {
        "kvmix_last_error": (C.c_char_p, []),
        "kvmix_abi_version": (i, []),
        "kvmix_launch_count": (u64, []),
        "kvmix_launch_count_of": (u64, [C.c_char_p]),
        "kvmix_packed_word_count": (sz, [sz, i]),
        "kvmix_feat_per_word": (i, [i, C.POINTER(C.c_int)]),
        "kvmix_pack": (i, [vp, sz, i, vp, vp]),
        "kvmix_unpack": (i, [vp, sz, i, vp, vp]),
        "kvmix_group_count": (sz, [i, i, i, i, i, i]),
        "kvmix_quantize": (i, [i, vp, i, i, i, i, i, i, i, vp, vp, vp]),
        "kvmix_dequantize": (i, [i, vp, vp, i, i, i, i, i, i, vp, vp]),
        "kvmix_config_validate": (i, [C.POINTER(LayerConfigC)]),
        "kvmix_rpc_target": (i, [i64, C.c_double, C.POINTER(C.c_int64)]),
        "kvmix_cache_create": (i, [C.POINTER(LayerConfigC), i, i, i, i64, i, C.POINTER(vp)]),
        "kvmix_cache_destroy": (None, [vp]),
        "kvmix_cache_set_shard": (i, [vp, i, i, i, i]),
        "kvmix_cache_reset": (i, [vp, vp]),
        "kvmix_cache_append": (i, [vp, vp, vp, i, i, vp]),
        "kvmix_cache_counters": (i, [vp, C.POINTER(C.c_int64)]),
        "kvmix_cache_shape": (i, [vp, C.POINTER(C.c_int64)]),
        "kvmix_cache_config": (i, [vp, C.POINTER(LayerConfigC)]),
        "kvmix_cache_memory_usage": (i, [vp, C.POINTER(MemoryReportC)]),
        "kvmix_cache_algorithmic_bytes": (i, [vp, C.POINTER(C.c_uint64)]),
        "kvmix_cache_snapshot": (i, [vp, vp, vp, vp]),
        "kvmix_cache_segment_info": (i, [vp, i, i, C.POINTER(C.c_int64)]),
        "kvmix_cache_export_segment": (i, [vp, i, i, vp, vp, vp]),
        "kvmix_cache_export_tail": (i, [vp, i, vp, vp]),
        "kvmix_cache_import_segment": (i, [vp, i, i, vp, vp, vp]),
        "kvmix_cache_import_tail": (i, [vp, i, vp, i64, vp]),
        "kvmix_attend": (i, [vp, vp, i, i, i, vp, C.POINTER(C.c_double), vp]),
        "kvmix_append_attend": (i, [vp, vp, vp, i, i, vp, i, i, i, vp, C.POINTER(C.c_double), vp]),
        "kvmix_attend_layers": (i, [C.POINTER(vp), i, C.POINTER(vp), i, i, i, C.POINTER(vp), vp]),
        "kvmix_append_attend_layers": (i, [C.POINTER(vp), i, C.POINTER(vp), C.POINTER(vp), i, i, C.POINTER(vp), i, i, i,
                                           C.POINTER(vp), vp]),
        "kvmix_fused_qk_scores": (i, [vp, vp, i, i, vp, vp]),
        "kvmix_softmax_rows": (i, [vp, i64, i64, vp]),
        "kvmix_fused_pv": (i, [vp, vp, i, vp, vp]),
        "kvmix_reference_attend": (i, [vp, vp, i, i, vp, vp, C.POINTER(C.c_double), vp]),
        "kvmix_scratch_reset": (None, []),
        "kvmix_scratch_allocated": (u64, []),
        "kvmix_set_knob": (i, [C.c_char_p, i]),
    }
    for name, (res, args) in sigs.items():
        fn = getattr(L, name)
        fn.restype = res
        fn.argtypes = args
    return L


def lib():
    """The loaded library. Builds it in-tree if the sources are newer (dev convenience)."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise ImportError(
                f"libkvmix_b200.so not found at {LIB_PATH}: run `python -m paper_2506_08018_b200.build` "
                "(there is no CPU fallback)")
        _lib = _declare(C.CDLL(LIB_PATH))
        if _lib.kvmix_abi_version() != 1:
            raise ImportError("libkvmix_b200.so ABI version mismatch")
    return _lib


def check(status: int) -> None:
    if status != OK:
        msg = lib().kvmix_last_error().decode(errors="replace")
        raise _ERRORS.get(status, KvmixError)(msg)


def launch_count() -> int:
    return int(lib().kvmix_launch_count())


def set_knob(name: str, value: int) -> None:
    """Override one kernel tuning/test knob (kvmix_set_knob)."""
    check(lib().kvmix_set_knob(name.encode(), int(value)))


def scratch_reset() -> None:
    lib().kvmix_scratch_reset()


def scratch_allocated() -> int:
    """Bytes of attention scratch requested since scratch_reset() (scratch.hpp:14-21)."""
    return int(lib().kvmix_scratch_allocated())


def tensor_core_launches() -> int:
    """Launches of the tensor-core attention kernels (warp-specialized or single-warp IMMA;
    attend_tc_kernel is always followed by an attend_mma_kernel window launch)."""
    return launch_count_of("attend_ws_kernel") + launch_count_of("attend_mma_kernel")


def launch_count_of(kernel: str) -> int:
    """Launches of one device kernel by name (which path served a call)."""
    return int(lib().kvmix_launch_count_of(kernel.encode()))
