"""Loader for ``libsfsketch_cuda.so`` (the C ABI in ``include/sfsketch_cuda.h``).

The library is built in-tree (``csrc/Makefile`` -> ``_lib/``). There is no
CPU fallback: every sketch operation goes through this library, and using a
sketch without a CUDA device or without the built library raises
``RuntimeError`` naming what is missing.
"""

from __future__ import annotations

import ctypes
import os
import subprocess

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("SFK_LIB_PATH") or os.path.join(_HERE, "_lib", "libsfsketch_cuda.so")  # env: A/B builds
CSRC = os.path.join(_HERE, "csrc")

KEY_U64, KEY_U32, KEY_RECORD = 0, 1, 2
OK, PHANTOM, SATURATED, UNSUPPORTED, BAD_OPCODE = 0, 1, 2, 3, 4
VARIANT_CODE = {"sf1": 1, "sf2": 2, "sf3": 3, "sf4": 4, "sff": 6}
FLAG_SEQUENTIAL = 1
# sfk_host_query_config keys and wire formats (include/sfsketch_cuda.h)
HQ_CHUNK, HQ_WIRE, HQ_DIRECT, HQ_THREADS, HQ_RING, HQ_LAST_WIRE = 0, 1, 2, 3, 4, 5
WIRE_AUTO, WIRE_I64, WIRE_U32, WIRE_C16 = 0, 1, 2, 3

# every symbol the header declares; tests check the built library exports them
EXPORTS = (
    "sfk_abi_version",
    "sfk_last_error",
    "sfk_stream_sync",
    "sfk_mix_batch",
    "sfk_load_keys",
    "sfk_min_query",
    "sfk_min_query_host",
    "sfk_min_query_host_staged",
    "sfk_host_query_config",
    "sfk_cm_workspace_size",
    "sfk_cm_apply",
    "sfk_cm_delta",
    "sfk_cu_workspace_size",
    "sfk_cu_apply",
    "sfk_sf_workspace_size",
    "sfk_sf_apply",
    "sfk_oracle_workspace_size",
    "sfk_oracle_slim_apply",
    "sfk_count_workspace_size",
    "sfk_count_apply",
    "sfk_count_query",
    "sfk_cml_workspace_size",
    "sfk_cml_apply",
    "sfk_cml_query",
    "sfk_pcg64_draws",
    "sfk_pcg64_bounded_workspace_size",
    "sfk_pcg64_bounded",
    "sfk_interleave_workspace_size",
    "sfk_interleave_deletions",
    "sfk_trace_workspace_size",
    "sfk_trace_parse_lines",
    "sfk_trace_compact",
    "sfk_launch_count",
    "sfk_gen_query_keys",
    "sfk_engine_stats",
    "sfk_engine_timing",
    "sfk_engine_last_ms",
    "sfk_engine_trace",
    "sfk_query_path",
    "sfk_small_batch_ops",
    "sfk_warp_batch_ops",
    "sfk_block_batch_ops",
    "sfk_blk_profile",
    "sfk_query_last_path",
    "sfk_query_index",
    "sfk_min_query_idx",
)

_lib = None


def build(jobs: int = 4) -> str:
    """Compile the CUDA sources for sm_100a (nvcc cross-compiles; no GPU needed)."""
    subprocess.run(["make", "-s", f"-j{jobs}", "-C", CSRC], check=True)
    return LIB_PATH


def load_library() -> ctypes.CDLL:
    """Load and type the library without touching a GPU."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        raise RuntimeError(
            f"libsfsketch_cuda.so is not built ({LIB_PATH}); run `make -C {CSRC}` or __graft_entry__.build()"
        )
    L = ctypes.CDLL(LIB_PATH)
    P, I, I64, SZ = ctypes.c_void_p, ctypes.c_int, ctypes.c_int64, ctypes.c_size_t
    L.sfk_abi_version.restype = I
    L.sfk_last_error.restype = ctypes.c_char_p
    L.sfk_stream_sync.argtypes = [P]
    L.sfk_mix_batch.argtypes = [P, I64, P, P]
    L.sfk_load_keys.argtypes = [P, I, I, I64, P, P]
    L.sfk_min_query.argtypes = [P, P, I, I64, P, I, I, I64, P, P]
    L.sfk_min_query_host.argtypes = [P, P, I, I64, P, I, I, I64, P, P]
    L.sfk_min_query_host_staged.argtypes = [P, P, I, I64, P, I, I, I64, P, P, I64, P]
    L.sfk_host_query_config.argtypes = [I, I64]
    L.sfk_host_query_config.restype = I64
    L.sfk_cm_workspace_size.argtypes = [I, I64, I64]
    L.sfk_cm_workspace_size.restype = SZ
    L.sfk_cu_workspace_size.argtypes = [I, I64, I64]
    L.sfk_cu_workspace_size.restype = SZ
    apply_args = [P, P, I, I64, P, P, I, I, I64, P, P, P, SZ, I, P]
    L.sfk_cm_apply.argtypes = apply_args
    L.sfk_cu_apply.argtypes = apply_args
    L.sfk_cm_delta.argtypes = [P, P, I, I64, P, P, I, I, I64, P]
    L.sfk_sf_workspace_size.argtypes = [I, I, I64, I64, I, I64]
    L.sfk_sf_workspace_size.restype = SZ
    L.sfk_sf_apply.argtypes = [I, P, P, P, P, P, I, I64, I64, I, P, P, I, I, I64, P, P, P, SZ, I, P]
    L.sfk_oracle_workspace_size.argtypes = [I, I64, I64]
    L.sfk_oracle_workspace_size.restype = SZ
    L.sfk_oracle_slim_apply.argtypes = [P, P, I, I64, P, I, I, P, I64, P, P, P, SZ, I, P]
    L.sfk_count_workspace_size.argtypes = [I, I64, I64]
    L.sfk_count_workspace_size.restype = SZ
    L.sfk_count_apply.argtypes = [P, P, I, I64, P, P, I, I, I64, P, P, SZ, I, P]
    L.sfk_count_query.argtypes = [P, P, I, I64, P, I, I, I64, P, P]
    L.sfk_cml_workspace_size.argtypes = [I, I64, I64]
    L.sfk_cml_workspace_size.restype = SZ
    L.sfk_cml_apply.argtypes = [P, P, I, I64, P, P, I, I, I64, P, ctypes.c_uint64, I64, P, P, SZ, I, P]
    L.sfk_cml_query.argtypes = [P, P, I, I64, P, I, I, I64, P, P, P]
    U64 = ctypes.c_uint64
    L.sfk_pcg64_draws.argtypes = [U64, U64, U64, U64, I64, I64, P, I64, P, P, P]
    L.sfk_pcg64_bounded_workspace_size.argtypes = [I64, I64]
    L.sfk_pcg64_bounded_workspace_size.restype = SZ
    L.sfk_pcg64_bounded.argtypes = [U64, U64, U64, U64, I64, I64, I64, P, P, P, SZ, P]
    L.sfk_interleave_workspace_size.argtypes = [I64]
    L.sfk_interleave_workspace_size.restype = SZ
    L.sfk_interleave_deletions.argtypes = [P, P, P, ctypes.c_double, I64, I64, P, P, P, SZ, P]
    L.sfk_trace_workspace_size.argtypes = [I64]
    L.sfk_trace_workspace_size.restype = SZ
    L.sfk_trace_parse_lines.argtypes = [P, I64, P, P, P, P, P, P, SZ, P]
    L.sfk_trace_compact.argtypes = [P, P, P, I64, P, P, P, P, SZ, I64, P]
    L.sfk_launch_count.restype = ctypes.c_ulonglong
    L.sfk_engine_stats.argtypes = [P, I]
    L.sfk_engine_timing.argtypes = [I]
    L.sfk_engine_last_ms.restype = ctypes.c_float
    L.sfk_engine_trace.argtypes = [P, SZ]
    L.sfk_query_path.argtypes = [I]
    L.sfk_small_batch_ops.argtypes = [I64]
    L.sfk_small_batch_ops.restype = I64
    L.sfk_warp_batch_ops.argtypes = [I64]
    L.sfk_warp_batch_ops.restype = I64
    L.sfk_block_batch_ops.argtypes = [I64]
    L.sfk_block_batch_ops.restype = I64
    L.sfk_blk_profile.argtypes = [P]
    L.sfk_query_index.argtypes = [P, I, I64, P, I, I, I64, P, P]
    L.sfk_min_query_idx.argtypes = [P, I, I64, P, I64, P, P]
    L.sfk_gen_query_keys.argtypes = [ctypes.c_uint64, P, P, ctypes.c_uint32, P, I64, I64, P, P]
    _lib = L
    return L


_cuda_ok = False


def lib() -> ctypes.CDLL:
    """The library, after checking (once) that a CUDA device is usable."""
    global _cuda_ok
    if not _cuda_ok:
        import torch

        if not torch.cuda.is_available():
            raise RuntimeError("paper_1701_04148_b200 needs a CUDA device (B200, sm_100a); no CPU fallback exists")
        _cuda_ok = True
    return load_library()


def check(rc: int, what: str) -> None:
    if rc != 0:
        msg = load_library().sfk_last_error().decode(errors="replace")
        raise RuntimeError(f"{what} failed (code {rc}): {msg}")


def stream_ptr(stream=None) -> int:
    """The raw cudaStream_t of `stream`, or of the current stream (the raw
    getter skips building a torch.cuda.Stream object: ~3 us per call)."""
    import torch

    if stream is not None:
        return int(stream.cuda_stream)
    try:
        return int(torch._C._cuda_getCurrentRawStream(torch._C._cuda_getDevice()))
    except AttributeError:  # older torch
        return int(torch.cuda.current_stream().cuda_stream)
