"""ctypes binding of libmpx.so (the C ABI declared in include/mpx.h).

The shared library is built in-tree (``__graft_entry__.build()``). There is
no CPU fallback: if the library is missing or a call fails the product path
raises ``MpxError``. Tensors cross the ABI as raw device pointers; the
launching stream is torch's current CUDA stream.

Dry runs (``DemandCounter`` sessions, preprocessing.py:369-403) allocate
``meta`` tensors; every wrapper skips the launch when its output is meta, so
the same protocol code sizes the dealer material without touching a GPU.
"""

from __future__ import annotations

import ctypes
import os

import torch

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("MPX_LIB") or os.path.join(_HERE, "libmpx.so")  # MPX_LIB: A/B builds

_P = ctypes.c_void_p
_I = ctypes.c_int
_L = ctypes.c_int64
_U = ctypes.c_uint64

_SIGS = {
    "mpx_ring_lin": [_P, _P, _U, _P, _U, _U, _P, _L, _I, _L, _I, _I, _P],
    "mpx_ring_mul": [_P, _P, _P, _L, _I, _P],
    "mpx_ring_rowdot": [_P, _P, _P, _I, _L, _L, _I, _P],
    "mpx_encode": [_P, _P, _L, _I, _I, _P],
    "mpx_decode": [_P, _P, _L, _I, _I, _P],
    "mpx_to_signed": [_P, _P, _L, _I, _P],
    "mpx_open_sum": [_P, _P, _I, _L, _I, _P],
    "mpx_open_xor": [_P, _P, _I, _L, _P],
    "mpx_mask_sub": [_P, _P, _P, _L, _I, _L, _I, _P],
    "mpx_trunc_sub_multi": [_P, _I, _I, _I, _P],
    "mpx_trunc_rows_bias": [_P, _P, _P, _I, _P, _L, _P, _L, _I, _L, _L, _L, _I, _I, _I, _U, _U, _I, _P],
    "mpx_trunc_expand_rows": [_P, _P, _P, _L, _P, _L, _I, _L, _L, _L, _L, _L, _I, _I, _U, _U, _I, _P],
    "mpx_mask_sub_t": [_P, _P, _L, _L, _P, _L, _L, _I, _L, _L, _L, _I, _P],
    "mpx_mask_sub_bs": [_P, _P, _L, _L, _P, _L, _L, _I, _L, _L, _I, _P],
    "mpx_mul_finish": [_P, _P, _P, _P, _P, _P, _L, _I, _L, _I, _I, _P],
    "mpx_mul_fused": [_P, _P, _P, _P, _P, _P, _L, _I, _L, _I, _I, _P],
    "mpx_trunc_mask": [_P, _P, _P, _L, _P, _L, _I, _L, _I, _I, _U, _I, _P],
    "mpx_trunc_finish": [_P, _P, _P, _L, _I, _L, _I, _I, _U, _I, _P],
    "mpx_trunc_fused": [_P, _P, _P, _L, _P, _L, _I, _L, _I, _I, _U, _U, _I, _P],
    "mpx_and_mask": [_P, _P, _P, _P, _P, _P, _L, _L, _I, _L, _I, _P],
    "mpx_and_finish": [_P, _P, _P, _P, _P, _P, _L, _L, _I, _L, _I, _I, _P],
    "mpx_carry_mask": [_P, _P, _P, _P, _P, _P, _P, _P, _L, _L, _I, _L, _I, _I, _I, _P],
    "mpx_carry_finish": [_P, _P, _P, _P, _P, _P, _P, _P, _P, _L, _L, _I, _L, _I, _I, _I, _I, _P],
    "mpx_carry_fused": [_P, _P, _P, _P, _P, _L, _L, _I, _L, _I, _I, _I, _I, _P],
    "mpx_pubadd_init": [_P, _P, _P, _P, _P, _P, _L, _L, _I, _L, _I, _I, _P],
    "mpx_sum_from_carries": [_P, _P, _P, _I, _L, _I, _P],
    "mpx_lmo_mask": [_P, _P, _P, _P, _P, _L, _L, _I, _L, _I, _I, _P],
    "mpx_lmo_finish": [_P, _P, _P, _P, _P, _P, _L, _L, _I, _L, _I, _I, _I, _P],
    "mpx_lmo_fused": [_P, _P, _P, _P, _L, _L, _I, _L, _I, _I, _I, _P],
    "mpx_bit2a_mask": [_P, _P, _P, _L, _L, _I, _L, _I, _P],
    "mpx_bit2a_finish": [_P, _P, _P, _L, _I, _L, _I, _I, _I, _P, _I, _P],
    "mpx_bits_op": [_P, _P, _P, _I, _I, _L, _I, _I, _I, _P],
    "mpx_bits_gather": [_P, _P, _P, _I, _L, _P],
    "mpx_bits_pack": [_P, _P, _L, _I, _P],
    "mpx_bits_unpack": [_P, _P, _L, _I, _P],
    "mpx_bits_flat_to_rows": [_P, _P, _L, _L, _I, _P],
    "mpx_bits_rows_to_flat": [_P, _P, _L, _I, _P],
    "mpx_gemm": [_P, _P, _P, _L, _L, _L, _L, _L, _L, _L, _I, _I, _P],
    "mpx_gemm_simt": [_P, _P, _P, _L, _L, _L, _L, _L, _L, _L, _I, _I, _P],
    "mpx_im2col": [_P, _P, _I, _L, _I, _I, _I, _I, _I, _I, _P],
    "mpx_col2im": [_P, _P, _I, _L, _I, _I, _I, _I, _I, _I, _I, _P],
    "mpx_limb_split": [_P, _P, _L, _L, _L, _L, _L, _L, _I, _P],
    "mpx_beaver_limbs": [_P, _P, _P, _P, _P, _L, _P, _L, _I, _L, _L, _L, _L, _L, _L, _I, _P],
    "mpx_beaver_gemm": [_P, _L, _P, _L, _P, _P, _P, _L, _P, _L, _I, _L, _L, _L, _I, _I, _P],
    "mpx_beaver_gemm_batched": [_P, _L, _L, _P, _L, _L, _P, _P, _P, _L, _L, _P, _L, _L, _I, _L, _L, _L, _L, _I, _I,
                                _P],
    "mpx_beaver_gemm_sim": [_P, _L, _L, _P, _L, _L, _P, _L, _L, _L, _L, _P, _L, _L, _P, _L, _L, _L, _L, _P, _L, _L,
                            _I, _L, _L, _L, _L, _I, _I, _P],
    "mpx_ring_colsum": [_P, _P, _I, _L, _L, _I, _P],
    "mpx_ring_pool_sum": [_P, _P, _L, _L, _L, _L, _L, _I, _P],
    "mpx_ring_pool_scatter": [_P, _P, _L, _L, _L, _L, _L, _I, _P],
    "mpx_ring_add_rowvec": [_P, _P, _I, _L, _L, _I, _I, _P],
    "mpx_gemm_limbs": [_P, _P, _P, _L, _L, _L, _L, _L, _L, _L, _L, _I, _I, _I, _P, _L, _P],
    "mpx_gemm_limbs_split": [_P, _P, _P, _P, _P, _L, _L, _L, _L, _L, _L, _L, _L, _I, _I, _P, _L, _I, _L, _P],
    "mpx_mask_limbs": [_P, _P, _P, _L, _L, _L, _P, _L, _L, _L, _I, _L, _L, _L, _L, _I, _I, _I, _I, _L, _L, _P],
    "mpx_mask_limbs2": [_P, _P, _P, _L, _L, _L, _P, _L, _L, _L, _L, _L, _P, _P, _P, _L, _L, _L, _P, _L, _L, _L,
                        _L, _L, _I, _L, _L, _I, _I, _I, _L, _L, _L, _L, _P],
    "mpx_philox_elems": [_P, _U, _U, _L, _L, _I, _P],
    "mpx_philox_bits": [_P, _U, _U, _L, _L, _P],
    "mpx_deal_share_arith": [_P, _L, _P, _U, _U, _L, _L, _I, _I, _I, _I, _P],
    "mpx_deal_share_bits": [_P, _L, _P, _U, _U, _L, _L, _I, _I, _I, _P],
    "mpx_philox_elems_dk": [_P, _P, _L, _L, _I, _P],
    "mpx_philox_bits_dk": [_P, _P, _L, _L, _P],
    "mpx_deal_share_arith_dk": [_P, _L, _P, _P, _L, _L, _I, _I, _I, _I, _P],
    "mpx_deal_share_bits_dk": [_P, _L, _P, _P, _L, _L, _I, _I, _I, _P],
    "mpx_beaver_tc_thin": [_P, _L, _P, _L, _P, _L, _L, _L, _P, _L, _P, _L, _L, _L, _P, _L, _I, _L, _L, _L, _I, _I,
                           _P],
    "mpx_beaver_tc_long": [_P, _L, _P, _L, _P, _L, _L, _L, _P, _L, _P, _L, _L, _L, _P, _L, _I, _L, _L, _L, _I, _I,
                           _P, _L, _P],
    "mpx_philox_probe": [_P, _L, _L, _P],
    "mpx_deal_triple": [_P, _P, _P, _L, _U, _U, _P, _L, _I, _I, _I, _I, _P],
    "mpx_deal_gen_arith": [_P, _L, _P, _U, _U, _P, _L, _L, _L, _I, _I, _I, _I, _I, _P],
    "mpx_deal_bintriple": [_P, _P, _P, _L, _U, _U, _P, _L, _I, _I, _I, _P],
    "mpx_deal_dabit": [_P, _L, _P, _L, _U, _U, _P, _L, _I, _I, _I, _I, _P],
    "mpx_deal_edabit_bits": [_P, _L, _U, _U, _P, _L, _L, _I, _I, _I, _I, _I, _P],
}

# entry points without a stream argument (bound with their own argtypes)
_PLAIN = {"mpx_last_cuda_error": ([], ctypes.c_int), "mpx_device_sm_count": ([_I], ctypes.c_int),
          "mpx_version": ([], ctypes.c_char_p), "mpx_cuda_error_string": ([_I], ctypes.c_char_p)}

BITS_XOR, BITS_AND, BITS_AND_PUB, BITS_XOR_PUB, BITS_XOR_SHR1, BITS_PARITY, BITS_SIGNFOLD, \
    BITS_SHL_OR, BITS_BCAST_PUB = range(9)


class MpxError(RuntimeError):
    """A libmpx call failed (bad argument or CUDA error)."""


_lib = None


def exported_symbols() -> list[str]:
    return sorted(list(_SIGS) + list(_PLAIN) + ["mpx_reciprocal_fused",
                                 "mpx_exp_fused", "mpx_log_fused", "mpx_fused_abi_sizes",
                                 "mpx_relu_fused", "mpx_maxlevel_fused", "mpx_attexp_fused",
                                 "mpx_maxtour_fused", "mpx_fused_tour_size", "mpx_softmax_fused",
                                 "mpx_fused_softmax_size"])


def load() -> ctypes.CDLL:
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        raise MpxError(f"{LIB_PATH} is missing: build it with __graft_entry__.build() "
                       "(the B200 path has no CPU fallback)")
    lib = ctypes.CDLL(LIB_PATH)
    for name, args in _SIGS.items():
        fn = getattr(lib, name)
        fn.argtypes = args
        fn.restype = ctypes.c_int
    for name, (args, res) in _PLAIN.items():
        fn = getattr(lib, name)
        fn.argtypes = args
        fn.restype = res
    _lib = lib
    return lib


def version() -> str:
    return load().mpx_version().decode()


def stream_ptr() -> int:
    return torch.cuda.current_stream().cuda_stream


def ptr(t) -> int | None:
    if t is None:
        return None
    return t.data_ptr()


# Launch accounting for the benchmark harness: LAUNCHES counts libmpx entry
# calls; between profile_begin() and profile_end() every call of the calling
# thread is bracketed by CUDA events on its stream.
import threading

LAUNCHES = 0
_TLS = threading.local()


def profile_begin() -> None:
    _TLS.prof = []


def profile_end() -> list:
    out = getattr(_TLS, "prof", None) or []
    _TLS.prof = None
    return out


def profiling() -> list | None:
    return getattr(_TLS, "prof", None)


def call(name: str, *args) -> None:
    """Invoke one libmpx entry point; raise MpxError on a non-zero return."""
    global LAUNCHES
    lib = load()
    LAUNCHES += 1
    prof = getattr(_TLS, "prof", None)
    if prof is not None:
        ev0 = torch.cuda.Event(enable_timing=True)
        ev1 = torch.cuda.Event(enable_timing=True)
        ev0.record()
        rc = getattr(lib, name)(*args, stream_ptr())
        ev1.record()
        prof.append((name, args, ev0, ev1))
    else:
        rc = getattr(lib, name)(*args, stream_ptr())
    check(name, rc)


MPX_OK, MPX_ERR_ARG, MPX_ERR_CUDA = 0, -1, -2


def check(name: str, rc: int) -> None:
    """Map a libmpx return code to the Python error behaviour: MPX_ERR_ARG
    (a shape / width / pointer precondition, the C side of the reference's
    ValueError) and MPX_ERR_CUDA both raise ``MpxError``."""
    if rc == MPX_OK:
        return
    lib = load()
    if rc == MPX_ERR_CUDA:
        code = lib.mpx_last_cuda_error()
        msg = lib.mpx_cuda_error_string(code).decode()
        raise MpxError(f"{name}: CUDA error {code} ({msg})")
    raise MpxError(f"{name}: returned {rc} (invalid argument)")


def device_sm_count(device: int | None = None) -> int:
    """SM count of the device (148 on B200), queried through libmpx."""
    dev = torch.cuda.current_device() if device is None else device
    n = load().mpx_device_sm_count(dev)
    if n <= 0:
        raise MpxError(f"mpx_device_sm_count({dev}) failed ({n})")
    return n


def is_dry(*tensors) -> bool:
    return any(t is not None and t.is_meta for t in tensors)
