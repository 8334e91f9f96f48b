"""ctypes binding of the C ABI in include/acegpu.h (lib/libacegpu.so).

There is no CPU fallback: importing this module on a machine without the
built library, or creating a context without an sm_100 GPU, raises.
"""
from __future__ import annotations

import ctypes as C
import os
import threading

import numpy as np

LIB_PATH = os.environ.get("ACEGPU_LIB") or os.path.join(
    os.path.dirname(os.path.abspath(__file__)), "lib", "libacegpu.so")  # ACEGPU_LIB: A/B probes

OK, EINVAL, ECUDA, ENODEV = 0, -1, -2, -3

u8p = C.POINTER(C.c_uint8)
u32p = C.POINTER(C.c_uint32)
u64p = C.POINTER(C.c_uint64)
vp = C.c_void_p
u64 = C.c_uint64
ctxp = C.c_void_p

_SIGS = {
    "acegpu_last_error": (C.c_char_p, []),
    "acegpu_version": (C.c_char_p, []),
    "acegpu_create": (C.c_int, [C.c_int, C.POINTER(C.c_void_p)]),
    "acegpu_destroy": (None, [ctxp]),
    "acegpu_launch_count": (C.c_uint64, [ctxp]),
    "acegpu_set_phase_timing": (C.c_int, [ctxp, C.c_int]),
    "acegpu_phase_times": (C.c_int, [ctxp, C.POINTER(C.c_float)]),
    "acegpu_set_segmented": (C.c_int, [ctxp, C.c_int]),
    "acegpu_host_alloc": (C.c_void_p, [C.c_size_t]),
    "acegpu_host_free": (None, [C.c_void_p]),
    "acegpu_sha256_varlen": (C.c_int, [ctxp, vp, vp, u64, vp]),
    "acegpu_sha256_strided": (C.c_int, [ctxp, vp, u64, u64, u64, vp]),
    "acegpu_prove_public_inputs": (C.c_int, [ctxp, vp, u64, vp]),
    "acegpu_prove_txs": (C.c_int, [ctxp, vp, vp, vp, u64, vp]),
    "acegpu_verify_mock": (C.c_int, [ctxp, vp, u64, vp]),
    "acegpu_aggregate_pairs": (C.c_int, [ctxp, vp, vp, u64, vp]),
    "acegpu_aggregate_tree": (C.c_int, [ctxp, vp, u64, vp, u64p, u64p]),
    "acegpu_prove_block": (C.c_int, [ctxp, vp, vp, vp, u64, vp, vp, u64p, u64p]),
    "acegpu_build_fc": (C.c_int, [ctxp, vp, u64, vp, vp, vp]),
    "acegpu_verify_fc": (C.c_int, [ctxp, vp, vp, vp, vp, u64, vp, C.POINTER(C.c_int)]),
    "acegpu_merkle_root": (C.c_int, [ctxp, vp, u64, vp]),
    "acegpu_block_hash": (C.c_int, [ctxp, vp, vp]),
    "acegpu_attest_prove_certify": (C.c_int, [ctxp, vp, vp, vp, u64, vp, vp, u64, vp, vp, vp, vp,
                                              u64p, u64p]),
    "acegpu_attest_prove_certify_dev": (C.c_int, [ctxp, vp, vp, vp, vp, u64, vp, vp, u64, vp, vp,
                                                  vp, vp]),
    "acegpu_attest_prove_certify_async": (C.c_int, [ctxp, vp, vp, vp, vp, u64, vp, vp, u64, vp,
                                                    vp, vp, vp]),
    "acegpu_attest_prove_certify_graph": (C.c_int, [ctxp, vp, vp, vp, vp, u64, vp, vp, u64, vp,
                                                    vp, vp, vp]),
    "acegpu_shard_roots_dev": (C.c_int, [ctxp, vp, vp, vp, vp, u64, u64, C.c_uint32, vp, u64, vp,
                                         vp, vp, vp]),
    "acegpu_combine_roots_dev": (C.c_int, [ctxp, vp, vp, vp, u64, u64, vp, vp, vp]),
    "acegpu_attest_verify": (C.c_int, [ctxp, vp, vp, vp, u64, vp, u64, vp, vp]),
    "acegpu_attest_generate": (C.c_int, [ctxp, vp, vp, u64, vp, u64, vp, vp, vp, vp]),
    "acegpu_attest_generate_dev": (C.c_int, [ctxp, vp, vp, vp, u64, vp, vp, vp, vp, vp]),
    "acegpu_derive_attest_keys": (C.c_int, [ctxp, vp, vp, u64, vp]),
    "acegpu_witness_check": (C.c_int, [ctxp, vp, vp, vp, u64, vp]),
    "acegpu_build_witness": (C.c_int, [ctxp, vp, vp, u64, vp]),
    "acegpu_witness_xor": (C.c_int, [ctxp, vp, vp, vp, vp, u64, u64, vp]),
    "acegpu_sha256_peak": (C.c_int, [ctxp, C.POINTER(C.c_double)]),
    "acegpu_sha256_probe": (C.c_int, [ctxp, C.c_int, C.c_int, C.c_uint32, C.POINTER(C.c_double)]),
    "acegpu_bn_field_batch": (C.c_int, [ctxp, C.c_int, C.c_int, vp, vp, u64, vp]),
    "acegpu_bn_convert_dev": (C.c_int, [ctxp, vp, C.c_int, vp, u64, C.c_int]),
    "acegpu_bn_ntt": (C.c_int, [ctxp, vp, C.c_uint32, C.c_int, C.c_int]),
    "acegpu_bn_ntt_dev": (C.c_int, [ctxp, vp, vp, vp, C.c_uint32, C.c_int, C.c_int]),
    "acegpu_bn_ntt3": (C.c_int, [ctxp, vp, C.c_uint32, C.c_int, C.c_int]),
    "acegpu_bn_ntt3_dev": (C.c_int, [ctxp, vp, vp, vp, C.c_uint32, C.c_int, C.c_int]),
    "acegpu_bn_scalar_muls": (C.c_int, [ctxp, C.c_int, vp, vp, u64, vp]),
    "acegpu_bn_msm_params": (C.c_int, [ctxp, C.POINTER(C.c_int), C.POINTER(C.c_int)]),
    "acegpu_bn_msm_prepare": (C.c_int, [ctxp, C.c_int, vp, u64, C.c_int, C.POINTER(C.c_void_p)]),
    "acegpu_bn_msm_prepare_vb": (C.c_int, [ctxp, C.c_int, vp, u64, C.c_int, u64,
                                           C.POINTER(C.c_void_p)]),
    "acegpu_bn_msm_free": (None, [C.c_void_p]),
    "acegpu_g16_setup_slice": (C.c_int, [ctxp, C.c_uint32, C.c_uint32, vp, C.c_uint32, C.c_uint32,
                                         vp, C.POINTER(C.c_void_p)]),
    "acegpu_g16_block_inputs_dev": (C.c_int, [ctxp, vp, C.c_void_p, vp, vp, vp, u64, vp, u64, vp,
                                              vp, vp, vp, vp, vp]),
    "acegpu_g16_prove_partial_dev": (C.c_int, [ctxp, vp, C.c_void_p, vp, vp, vp]),
    "acegpu_g16_prove_phase1_dev": (C.c_int, [ctxp, vp, C.c_void_p, vp, vp, C.c_int, vp]),
    "acegpu_g16_prove_phase2_dev": (C.c_int, [ctxp, vp, C.c_void_p, vp, vp]),
    "acegpu_g16_finish_dev": (C.c_int, [ctxp, vp, C.c_void_p, vp, C.c_uint32, vp, vp, vp, vp]),
    "acegpu_bn_msm_run": (C.c_int, [ctxp, C.c_void_p, vp, vp]),
    "acegpu_bn_msm_run_dev": (C.c_int, [ctxp, vp, C.c_void_p, vp, vp]),
    "acegpu_g16_setup": (C.c_int, [ctxp, C.c_uint32, C.c_uint32, vp, C.POINTER(C.c_void_p)]),
    "acegpu_g16_free": (None, [C.c_void_p]),
    "acegpu_r1cs_free": (None, [C.c_void_p]),
    "acegpu_witprog_free": (None, [C.c_void_p]),
    "acegpu_witprog_create": (C.c_int, [ctxp, vp, u64, vp, u64, C.c_uint32, vp, C.c_uint32,
                                        C.c_uint32, C.POINTER(C.c_void_p)]),
    "acegpu_witprog_run": (C.c_int, [ctxp, C.c_void_p, vp, vp, C.c_uint32, vp]),
    "acegpu_witprog_run_dev": (C.c_int, [ctxp, C.c_void_p, C.c_void_p, vp, u64, vp, C.c_uint32,
                                         C.c_uint32, vp]),
    "acegpu_r1cs_shape": (C.c_int, [C.c_void_p, C.POINTER(u64), C.POINTER(u64), C.POINTER(u64)]),
    "acegpu_g16_shape": (C.c_int, [C.c_void_p, u64p, u64p, C.POINTER(C.c_uint32)]),
    "acegpu_g16_domain": (C.c_int, [C.c_void_p, u64p]),
    "acegpu_g16_prove_chunk": (C.c_int, [ctxp, C.c_void_p, vp, vp, vp, vp, vp, vp]),
    "acegpu_g16_prove_chunk_dev": (C.c_int, [ctxp, vp, C.c_void_p, vp, vp, vp, vp, vp, vp]),
    "acegpu_g16_vk": (C.c_int, [ctxp, C.c_void_p, vp]),
    "acegpu_g16_verify_batch": (C.c_int, [ctxp, C.c_void_p, vp, vp, u64, C.POINTER(C.c_int)]),
    "acegpu_r1cs_create": (C.c_int, [ctxp, u64, u64, u64, vp, vp, vp, C.POINTER(C.c_void_p)]),
    "acegpu_r1cs_eval": (C.c_int, [ctxp, C.c_void_p, vp, vp, vp, vp]),
    "acegpu_g16_setup_r1cs": (C.c_int, [ctxp, C.c_void_p, vp, C.POINTER(C.c_void_p)]),
    "acegpu_g16_prove_z": (C.c_int, [ctxp, C.c_void_p, vp, vp, vp, vp, vp]),
    "acegpu_g16_prove_z_dev": (C.c_int, [ctxp, C.c_void_p, C.c_void_p, vp, vp, vp, vp, vp]),
    "acegpu_g16_prove_block": (C.c_int, [ctxp, C.c_void_p, vp, vp, vp, u64, vp, vp, u64, vp, vp,
                                         vp, vp, vp, vp]),
    "acegpu_g16_verify_batch_seed": (C.c_int, [ctxp, C.c_void_p, vp, vp, u64, C.POINTER(C.c_int),
                                               vp]),
    "acegpu_g16_verify_fc": (C.c_int, [ctxp, C.c_void_p, vp, vp, vp, vp, u64, vp, vp, u64p,
                                       C.POINTER(C.c_int)]),
    "acegpu_g16_shard_roots_dev": (C.c_int, [ctxp, vp, C.c_void_p, vp, vp, vp, u64, u64, vp, u64,
                                             vp, vp, vp, vp, vp]),
    "acegpu_bn_pairing": (C.c_int, [ctxp, u64, vp, vp, vp, C.POINTER(C.c_int)]),
    "acegpu_bn_f12_op": (C.c_int, [ctxp, C.c_int, vp, vp]),
    "acegpu_light_check": (C.c_int, [ctxp, vp, vp, vp, u64, vp, u64, u64, u64, vp, u64p]),
    "acegpu_light_check_dev": (C.c_int, [ctxp, vp, vp, vp, vp, u64, vp, u64, u64, u64, vp, vp]),
    "acegpu_build_block_dev": (C.c_int, [ctxp, vp, vp, vp, vp, u64, vp, vp, vp, vp, vp, vp, u64p]),
    "acegpu_imad_peak": (C.c_int, [ctxp, C.POINTER(C.c_double)]),
    "acegpu_bn_mul_rate": (C.c_int, [ctxp, C.c_int, C.POINTER(C.c_double)]),
}


def load_library(path: str = LIB_PATH) -> C.CDLL:
    if not os.path.exists(path):
        raise ImportError(
            f"libacegpu.so not found at {path}; build it with "
            "`python -c 'import __graft_entry__ as g; g.build()'` (no CPU fallback exists)")
    lib = C.CDLL(path)
    for name, (res, args) in _SIGS.items():
        f = getattr(lib, name)
        f.restype = res
        f.argtypes = args
    return lib


_lib: C.CDLL | None = None
_lib_lock = threading.Lock()


def lib() -> C.CDLL:
    global _lib
    with _lib_lock:
        if _lib is None:
            _lib = load_library()
        return _lib


class AceGpuError(RuntimeError):
    pass


def check(rc: int) -> None:
    if rc == OK:
        return
    msg = lib().acegpu_last_error().decode(errors="replace")
    if rc == EINVAL:
        raise ValueError(msg)  # std::invalid_argument in the reference
    raise AceGpuError(f"acegpu error {rc}: {msg}")


def addr(x) -> int | None:
    """Address of a numpy array / bytes / ctypes buffer / torch tensor (or None)."""
    if x is None:
        return None
    if isinstance(x, np.ndarray):
        assert x.flags["C_CONTIGUOUS"]
        return x.ctypes.data
    if isinstance(x, (bytes, bytearray)):
        raise TypeError("pass numpy arrays (bytes objects are immutable / unaligned)")
    if hasattr(x, "data_ptr"):
        return x.data_ptr()
    return C.addressof(x)


def as_u8(b) -> np.ndarray:
    if isinstance(b, np.ndarray):
        return np.ascontiguousarray(b, dtype=np.uint8)
    return np.frombuffer(bytes(b), np.uint8).copy() if len(b) else np.zeros(1, np.uint8)


class Context:
    """One libacegpu context (one CUDA device, one stream, one workspace)."""

    def __init__(self, device: int = 0):
        self.lib = lib()
        h = C.c_void_p()
        check(self.lib.acegpu_create(int(device), C.byref(h)))
        self.h = h
        self.device = device
        self.lock = threading.Lock()

    def close(self) -> None:
        if self.h:
            self.lib.acegpu_destroy(self.h)
            self.h = None

    def __del__(self):  # pragma: no cover - interpreter shutdown ordering
        try:
            self.close()
        except Exception:
            pass

    @property
    def launches(self) -> int:
        return int(self.lib.acegpu_launch_count(self.h))

    def call(self, name: str, *args) -> None:
        """Arrays / tensors may be passed directly: they stay referenced (alive)
        for the duration of the call, unlike a bare ``addr(temporary)``."""
        conv = [addr(a) if isinstance(a, np.ndarray) or hasattr(a, "data_ptr") else a
                for a in args]
        check(getattr(self.lib, name)(self.h, *conv))


_ctx: dict[int, Context] = {}
_ctx_lock = threading.Lock()


def default_device() -> int:
    env = os.environ.get("ACEGPU_DEVICE", os.environ.get("LOCAL_RANK"))
    return int(env) if env is not None else 0


def context(device: int | None = None) -> Context:
    dev = default_device() if device is None else device
    with _ctx_lock:
        if dev not in _ctx:
            _ctx[dev] = Context(dev)
        return _ctx[dev]
