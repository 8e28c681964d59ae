"""ctypes binding of the C-ABI library ``libff_chain.so`` (include/ff_chain.h).

The shared library is built in-tree by ``__graft_entry__.build()`` (or
``python -m paper_2512_12949_b200.build``).  There is no fallback: if the
library is missing, every GPU entry point raises :class:`NativeUnavailable`.
"""

from __future__ import annotations

import ctypes
import os
import threading

from .errors import CapacityExceeded, FusePlanError, PlanError

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("FF_CHAIN_LIB") or os.path.join(_HERE, "libff_chain.so")  # FF_CHAIN_LIB: A/B builds

FF_OK = 0
FF_ERR_PLAN = 1
FF_ERR_CAPACITY = 2
FF_ERR_UNSUPPORTED = 3
FF_ERR_CUDA = 4
FF_ERR_ARG = 5

KIND = {"standard_ffn": 0, "gated_ffn": 1}
ACT = {"identity": 0, "relu": 1, "silu": 2, "gelu": 3}
LOWERING = {"n/a": 0, "spatial_split": 1, "doubled_k": 2}
XCHG_DSM, XCHG_L2, XCHG_L2_PAIR, XCHG_L2_DSMR = 0, 1, 2, 3  # ff_chain.h FF_XCHG_*
DTYPE = {"bf16": 0, "f16": 1}

# Exported symbols (must match include/ff_chain.h).
EXPORTS = (
    "ff_plan_lower",
    "ff_plan_lower_ex",
    "ff_auto_config",
    "ff_auto_config_ex",
    "ff_chain_workspace_bytes",
    "ff_chain_launch",
    "ff_chain_run_plan",
    "ff_plan_workspace_bytes",
    "ff_chain_launch_debug",
    "ff_chain_kernel_count",
    "ff_config_deterministic",
    "ff_config_finish",
    "ff_set_profile_buffer",
    "ff_set_variant",
    "ff_last_error",
    "ff_version",
    "ff_conv_chain_desc",
    "ff_conv_chain_lower",
    "ff_conv_chain_workspace_bytes",
    "ff_conv_chain_launch",
)


class NativeUnavailable(RuntimeError):
    """The sm_100a extension is not built / cannot be loaded."""


class UnsupportedPlan(FusePlanError):
    """Structurally valid plan with no sm_100a lowering (FF_ERR_UNSUPPORTED)."""


class NativeError(FusePlanError):
    """CUDA runtime failure inside the native library (FF_ERR_CUDA / FF_ERR_ARG)."""


class ChainDesc(ctypes.Structure):
    _fields_ = [
        ("kind", ctypes.c_int32),
        ("activation", ctypes.c_int32),
        ("m", ctypes.c_int64),
        ("n", ctypes.c_int64),
        ("k", ctypes.c_int64),
        ("l", ctypes.c_int64),
        ("element_size", ctypes.c_int32),
        ("dtype", ctypes.c_int32),
    ]


class PlanDesc(ctypes.Structure):
    _fields_ = [
        ("spatial_mask", ctypes.c_uint32),
        ("temporal", ctypes.c_int32 * 4),
        ("n_temporal", ctypes.c_int32),
        ("block", ctypes.c_int64 * 4),
        ("cluster", ctypes.c_int32 * 4),
        ("gated_lowering", ctypes.c_int32),
    ]


class KernelConfig(ctypes.Structure):
    _fields_ = [
        ("ring", ctypes.c_int32),
        ("n_splits", ctypes.c_int32),
        ("nb", ctypes.c_int32),
        ("lb", ctypes.c_int32),
        ("exchange", ctypes.c_int32),
        ("m_tiles", ctypes.c_int32),
        ("l_clusters", ctypes.c_int32),
        ("steps", ctypes.c_int32),
        ("units", ctypes.c_int32),
        ("rings", ctypes.c_int32),
        ("grid_ctas", ctypes.c_int32),
    ]

    def as_dict(self) -> dict:
        return {name: int(getattr(self, name)) for name, _ in self._fields_}


class ConvDesc(ctypes.Structure):
    """ffConvDesc: ConvChainConfig (workload.py:168-184) + batch and activation."""

    _fields_ = [(name, ctypes.c_int32)
                for name in ("batch", "h", "w", "ic", "oc1", "oc2", "k1", "k2", "activation", "dtype")]


class Tensors(ctypes.Structure):
    _fields_ = [
        ("a", ctypes.c_void_p),
        ("b", ctypes.c_void_p),
        ("b1", ctypes.c_void_p),
        ("d", ctypes.c_void_p),
        ("e", ctypes.c_void_p),
    ]


_lib = None
_lock = threading.Lock()


def load(path: str = LIB_PATH):
    """Load (once) and return the native library; raises NativeUnavailable."""
    global _lib
    with _lock:
        if _lib is not None:
            return _lib
        if not os.path.exists(path):
            raise NativeUnavailable(
                f"{path} not found: build it with `python -c 'import __graft_entry__ as g; g.build()'`"
            )
        lib = ctypes.CDLL(path)
        P = ctypes.POINTER
        lib.ff_plan_lower.argtypes = [P(ChainDesc), P(PlanDesc), ctypes.c_int32, P(KernelConfig)]
        lib.ff_auto_config.argtypes = [P(ChainDesc), ctypes.c_int32, P(KernelConfig)]
        lib.ff_plan_lower_ex.argtypes = [P(ChainDesc), P(PlanDesc), ctypes.c_int32, ctypes.c_int32, P(KernelConfig)]
        lib.ff_auto_config_ex.argtypes = [P(ChainDesc), ctypes.c_int32, ctypes.c_int32, P(KernelConfig)]
        lib.ff_chain_workspace_bytes.argtypes = [P(ChainDesc), P(KernelConfig)]
        lib.ff_chain_workspace_bytes.restype = ctypes.c_size_t
        lib.ff_chain_launch.argtypes = [P(ChainDesc), P(KernelConfig), P(Tensors), ctypes.c_void_p,
                                        ctypes.c_size_t, ctypes.c_void_p]
        lib.ff_chain_run_plan.argtypes = [P(ChainDesc), P(PlanDesc), P(Tensors), ctypes.c_void_p,
                                          ctypes.c_size_t, ctypes.c_void_p]
        lib.ff_plan_workspace_bytes.argtypes = [P(ChainDesc), P(PlanDesc)]
        lib.ff_plan_workspace_bytes.restype = ctypes.c_size_t
        lib.ff_chain_launch_debug.argtypes = [P(ChainDesc), P(KernelConfig), P(Tensors), ctypes.c_void_p,
                                              ctypes.c_size_t, ctypes.c_void_p, ctypes.c_void_p]
        lib.ff_chain_kernel_count.argtypes = [P(ChainDesc), P(KernelConfig)]
        lib.ff_config_deterministic.argtypes = [P(ChainDesc), P(KernelConfig), ctypes.c_int32,
                                                P(ctypes.c_int32)]
        lib.ff_config_finish.argtypes = [P(ChainDesc), ctypes.c_int32, P(KernelConfig)]
        lib.ff_set_profile_buffer.argtypes = [ctypes.c_void_p]
        lib.ff_set_variant.argtypes = [ctypes.c_uint32]
        lib.ff_conv_chain_desc.argtypes = [P(ConvDesc), P(ChainDesc)]
        lib.ff_conv_chain_lower.argtypes = [P(ConvDesc), ctypes.c_int32, ctypes.c_int32, P(KernelConfig)]
        lib.ff_conv_chain_workspace_bytes.argtypes = [P(ConvDesc), P(KernelConfig)]
        lib.ff_conv_chain_workspace_bytes.restype = ctypes.c_size_t
        lib.ff_conv_chain_launch.argtypes = [P(ConvDesc), P(KernelConfig), P(Tensors), ctypes.c_void_p,
                                             ctypes.c_size_t, ctypes.c_void_p]
        lib.ff_last_error.restype = ctypes.c_char_p
        lib.ff_version.restype = ctypes.c_char_p
        _lib = lib
        return lib


def check(rc: int) -> None:
    """Map a C status code back to the reference exception classes."""
    if rc == FF_OK:
        return
    msg = load().ff_last_error().decode("utf-8", "replace")
    if rc == FF_ERR_PLAN:
        raise PlanError(msg)
    if rc == FF_ERR_CAPACITY:
        # the library reports "<tensor>:<floor tier>:<unplaced bytes>|<text>" (ff_chain.cu: fail_capacity)
        head, _, text = msg.partition("|")
        tensor, floor, unplaced = (head.split(":") + ["", "", "0"])[:3]
        exc = CapacityExceeded(tensor or "C", floor or "tmem", int(unplaced) if unplaced.isdigit() else 0)
        exc.args = (f"{exc.args[0]} ({text})",) if text else exc.args
        raise exc
    if rc == FF_ERR_UNSUPPORTED:
        raise UnsupportedPlan(msg)
    raise NativeError(f"native status {rc}: {msg}")
