"""ctypes binding of libkpm.so (the C-ABI declared in include/kpm.h).

The shared library is built in-tree (``paper_1905_09758_b200/libkpm.so``) by
``__graft_entry__.build()`` / ``make -C paper_1905_09758_b200/csrc``.  There is
no CPU fallback: if the library or a B200 is missing, every compute entry point
raises instead of silently running something else.
"""

from __future__ import annotations

import ctypes
import os
import threading

import numpy as np

from .errors import NetdosError, RecurrenceBlowupError

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("KPM_LIB") or os.path.join(HERE, "libkpm.so")

KPM_OK = 0
KPM_EINVAL = -1
KPM_ENONFINITE = -2
KPM_ENOMEM = -3
KPM_ECUDA = -4
KPM_EZEROMASS = -5
KPM_ENODEV = -6
KPM_PARSE_HASH_COMMENTS = 1

MODE_DOS_DOUBLING = 0
MODE_DOS_DIRECT = 1
MODE_LDOS = 2
LDOS_RAW = 1

_c_i64 = ctypes.c_int64
_c_i32 = ctypes.c_int32
_c_int = ctypes.c_int
_c_dbl = ctypes.c_double
_c_vp = ctypes.c_void_p
_c_u32 = ctypes.c_uint32
_c_u64 = ctypes.c_uint64
_PP = ctypes.POINTER(ctypes.c_void_p)

# name -> (restype, argtypes); the full export list of include/kpm.h
SIGNATURES = {
    "kpm_abi_version": (_c_int, []),
    "kpm_last_error": (ctypes.c_char_p, []),
    "kpm_device_count": (_c_int, [ctypes.POINTER(_c_int)]),
    "kpm_init": (_c_int, [_c_int, _PP]),
    "kpm_finalize": (None, [_c_vp]),
    "kpm_ctx_stream": (_c_vp, [_c_vp]),
    "kpm_ctx_synchronize": (_c_int, [_c_vp]),
    "kpm_device_alloc": (_c_int, [_c_vp, _c_i64, _PP]),
    "kpm_device_free": (_c_int, [_c_vp, _c_vp]),
    "kpm_memcpy": (_c_int, [_c_vp, _c_vp, _c_vp, _c_i64, _c_int]),
    "kpm_host_alloc": (_c_int, [_c_i64, _PP]),
    "kpm_host_free": (_c_int, [_c_vp]),
    "kpm_host_prefault": (_c_int, [_c_vp, _c_i64, _c_int]),
    "kpm_mem_info": (_c_int, [_c_vp, ctypes.POINTER(_c_i64), ctypes.POINTER(_c_i64)]),
    "kpm_graph_from_edges": (_c_int, [_c_vp, _c_i64, _c_vp, _c_vp, _c_i64, _c_int, _PP]),
    "kpm_graph_from_csr": (_c_int, [_c_vp, _c_i64, _c_vp, _c_vp, _c_i64, _c_vp, _c_dbl,
                                    _c_dbl, _PP]),
    "kpm_graph_from_csr32": (_c_int, [_c_vp, _c_i64, _c_vp, _c_vp, _c_i64, _c_vp, _c_dbl,
                                      _c_dbl, _PP]),
    "kpm_graph_prepare": (_c_int, [_c_vp, _c_i64, ctypes.POINTER(ctypes.c_int32)]),
    "kpm_graph_info": (_c_int, [_c_vp, ctypes.POINTER(_c_i64), ctypes.POINTER(_c_i64),
                                ctypes.POINTER(_c_i64)]),
    "kpm_graph_export": (_c_int, [_c_vp, _c_vp, _c_vp, _c_vp]),
    "kpm_graph_free": (None, [_c_vp]),
    "kpm_csr_matvec": (_c_int, [_c_vp, _c_i64, _c_vp, _c_vp, _c_vp, _c_i64, _c_vp, _c_i64,
                                _c_i64, _c_vp]),
    "kpm_probes_rademacher": (_c_int, [_c_vp, _c_i64, _c_i64, _c_vp, _c_vp, _c_i64, _c_i64]),
    "kpm_filter_probes": (_c_int, [_c_vp, _c_i64, _c_i64, _c_vp, _c_i64, _c_i64, _c_vp,
                                   _c_vp, _c_vp, _c_vp]),
    "kpm_run_create": (_c_int, [_c_vp, _c_i64, _c_i32, _c_i32, _c_i32, _PP]),
    "kpm_run_set_probes": (_c_int, [_c_vp, _c_vp, _c_i64]),
    "kpm_run_set_rademacher": (_c_int, [_c_vp, _c_vp]),
    "kpm_run_advance": (_c_int, [_c_vp, _c_i32, ctypes.POINTER(_c_i32)]),
    "kpm_run_total_steps": (_c_int, [_c_vp]),
    "kpm_run_set_timing": (_c_int, [_c_vp, _c_int]),
    "kpm_run_kernel_time": (_c_int, [_c_vp, ctypes.POINTER(_c_dbl), ctypes.POINTER(_c_i32)]),
    "kpm_run_result": (_c_int, [_c_vp, _c_vp, _c_dbl, ctypes.POINTER(_c_i64)]),
    "kpm_run_ldos_values": (_c_int, [_c_vp, _PP]),
    "kpm_run_accumulate": (_c_int, [_c_vp, _c_vp]),
    "kpm_run_trim": (_c_int, [_c_vp]),
    "kpm_graph_replicate": (_c_int, [_c_vp, _c_vp, _PP]),
    "kpm_run_block": (_c_int, [_c_vp, _PP, ctypes.POINTER(_c_i64), ctypes.POINTER(_c_i32)]),
    "kpm_run_free": (None, [_c_vp]),
    "kpm_dos_contrib": (_c_int, [_c_vp, _c_vp, _c_i64, _c_i32, _c_i32, _c_vp]),
    "kpm_ldos": (_c_int, [_c_vp, _c_vp, _c_i64, _c_i32, _c_i32, _c_dbl, _c_vp,
                          ctypes.POINTER(_c_i64)]),
    "kpm_rmat_edges": (_c_int, [_c_vp, _c_int, _c_u64, _c_u32, _c_u32, _c_u32, _c_i64, _c_i64,
                                _c_vp, _c_vp]),
    "kpm_graph_rmat": (_c_int, [_c_vp, _c_int, _c_i64, _c_u64, _c_u32, _c_u32, _c_u32, _PP]),
    "kpm_gen_preferential_attachment": (_c_int, [_c_i64, _c_i64, _c_vp, _c_vp, _c_vp]),
    "kpm_graph_from_csr_part": (_c_int, [_c_vp, _c_i64, _c_i64, _c_i64, _c_vp, _c_vp, _c_i64,
                                         _c_vp, _c_dbl, _c_dbl, _PP]),
    "kpm_graph_rmat_part": (_c_int, [_c_vp, _c_int, _c_i64, _c_u64, _c_u32, _c_u32, _c_u32,
                                     _c_i64, _c_i64, _PP]),
    "kpm_graph_part_info": (_c_int, [_c_vp, ctypes.POINTER(_c_i64), ctypes.POINTER(_c_i64)]),
    "kpm_graph_set_dinv": (_c_int, [_c_vp, _c_vp]),
    "kpm_run_blocks": (_c_int, [_c_vp, _PP, _PP]),
    "kpm_run_set_partition": (_c_int, [_c_vp, _c_int, _c_vp, _c_int, _c_vp, _c_vp]),
    "kpm_ipc_get_handle": (_c_int, [_c_vp, _c_vp]),
    "kpm_ipc_open_handle": (_c_int, [_c_vp, _c_vp, _PP]),
    "kpm_ipc_close": (_c_int, [_c_vp]),
    "kpm_motif_scan": (_c_int, [_c_vp] + [_c_vp] * 8),
    "kpm_parse_edges": (_c_int, [_c_vp, _c_vp, _c_i64, _c_i64, _c_int, _c_vp, _c_vp, _c_vp,
                                 _c_vp, _c_vp]),
    "kpm_edges_finalize": (_c_int, [_c_vp, _c_i64, _c_vp, _c_vp, _c_vp, _c_int, _c_i64,
                                    _c_vp, _c_vp, _c_vp, _c_vp, _c_vp, _c_vp]),
    "kpm_lanczos": (_c_int, [_c_vp, _c_vp, _c_i64, _c_i64, _c_i32, _c_vp, _c_vp, _c_vp, _c_vp,
                             _c_vp, _c_vp, _c_vp]),
    "kpm_ldos_histogram": (_c_int, [_c_vp, _c_vp, _c_i64, _c_i64, _c_i32, _c_vp, _c_vp, _c_i32,
                                    _c_vp, _c_vp, ctypes.POINTER(_c_dbl)]),
}

_lib = None
_lock = threading.RLock()


class KpmLibraryError(NetdosError, RuntimeError):
    """libkpm.so is missing, was built for another ABI, or no B200 is usable."""


def load():
    """Load libkpm.so (raises KpmLibraryError if it is absent)."""
    global _lib
    if _lib is not None:
        return _lib
    with _lock:
        if _lib is not None:
            return _lib
        if not os.path.exists(LIB_PATH):
            raise KpmLibraryError(
                f"{LIB_PATH} not built; run __graft_entry__.build() or "
                "`make -C paper_1905_09758_b200/csrc` (there is no CPU fallback)")
        lib = ctypes.CDLL(LIB_PATH)
        for name, (res, args) in SIGNATURES.items():
            fn = getattr(lib, name)
            fn.restype = res
            fn.argtypes = args
        if lib.kpm_abi_version() != 1:
            raise KpmLibraryError("libkpm ABI version mismatch")
        _lib = lib
    return _lib


def last_error() -> str:
    return load().kpm_last_error().decode(errors="replace")


def check(rc: int, what: str = "") -> None:
    """Map a libkpm status to the reference's exception types."""
    if rc == KPM_OK:
        return
    msg = last_error()
    if what:
        msg = f"{what}: {msg}"
    if rc == KPM_EINVAL or rc == KPM_EZEROMASS:
        raise ValueError(msg)
    if rc == KPM_ENONFINITE:
        raise RecurrenceBlowupError(msg)
    if rc == KPM_ENOMEM:
        raise MemoryError(msg)
    raise KpmLibraryError(f"libkpm status {rc}: {msg}")


def prefault(a, threads=0):
    """Page in a fresh host result array on host threads (kpm_host_prefault)
    so the D2H copy into it does not fault page by page; its contents are
    overwritten."""
    if a.nbytes:
        check(load().kpm_host_prefault(a.ctypes.data, a.nbytes, int(threads)),
              "host_prefault")
    return a


def ptr(a) -> int | None:
    """Raw address of a numpy array (or torch tensor / int) for ctypes."""
    if a is None:
        return None
    if isinstance(a, int):
        return a
    if isinstance(a, np.ndarray):
        return a.ctypes.data
    if hasattr(a, "data_ptr"):
        return a.data_ptr()
    raise TypeError(f"cannot take the address of {type(a)!r}")


class Context:
    """A libkpm context: one GPU and its own CUDA stream.  ``get(device)`` is
    the process's shared context of a device; ``pool`` adds further contexts
    (their own streams) when a device is listed more than once."""

    _by_key: dict[tuple[int, int], "Context"] = {}

    def __init__(self, device: int = 0):
        lib = load()
        h = ctypes.c_void_p()
        check(lib.kpm_init(int(device), ctypes.byref(h)), "kpm_init")
        self.device = int(device)
        self.handle = h.value

    @classmethod
    def get(cls, device: int | None = None, slot: int = 0) -> "Context":
        if device is None:
            device = default_device()
        key = (int(device), int(slot))
        with _lock:
            ctx = cls._by_key.get(key)
            if ctx is None:
                ctx = cls(device)
                cls._by_key[key] = ctx
        return ctx

    @classmethod
    def pool(cls, devices) -> list["Context"]:
        """Contexts for a device list; a repeated device gets another slot."""
        seen: dict[int, int] = {}
        out = []
        for d in devices:
            k = seen.get(int(d), 0)
            seen[int(d)] = k + 1
            out.append(cls.get(int(d), k))
        return out

    @property
    def stream(self) -> int:
        return load().kpm_ctx_stream(self.handle)

    def synchronize(self) -> None:
        check(load().kpm_ctx_synchronize(self.handle), "synchronize")

    def mem_info(self):
        f, t = ctypes.c_int64(), ctypes.c_int64()
        check(load().kpm_mem_info(self.handle, ctypes.byref(f), ctypes.byref(t)), "mem_info")
        return f.value, t.value


def default_device() -> int:
    """LOCAL_RANK under torchrun, else KPM_DEVICE, else 0."""
    for var in ("KPM_DEVICE", "LOCAL_RANK"):
        v = os.environ.get(var)
        if v not in (None, ""):
            return int(v)
    return 0


def devices_for(threads=1) -> list[int]:
    """GPUs one moment call uses (the reference's ``threads``
    knob, kpm.py:92-93 / NETDOS_THREADS cli.py:31-35, maps to a GPU count).
    KPM_DEVICES ("0,1,...", "all"; a repeated id adds a context on that GPU)
    wins; under torchrun (LOCAL_RANK set) a process keeps its own GPU; else
    ``threads`` > 1 uses min(threads, visible GPUs) starting at the default
    device."""
    env = os.environ.get("KPM_DEVICES", "").strip()
    if env:
        if env == "all":
            return list(range(device_count()))
        return [int(x) for x in env.split(",") if x.strip()]
    first = default_device()
    if os.environ.get("LOCAL_RANK") not in (None, "") or int(threads or 1) <= 1:
        return [first]
    count = device_count()
    want = min(int(threads), count)
    return [(first + i) % count for i in range(want)]


def device_count() -> int:
    c = ctypes.c_int(0)
    check(load().kpm_device_count(ctypes.byref(c)))
    return c.value
