"""ctypes binding of libhimeno_b200.so (C ABI: include/himeno_b200.h).

The library is the product's compute path; there is no Python or CPU
fallback for it.  ``load()`` raises ``NativeUnavailable`` when the .so is
missing or has the wrong ABI version, and context creation raises
``DeviceError`` when no CUDA device is present.
"""

from __future__ import annotations

import ctypes as C
import os
import threading
from pathlib import Path

from .errors import DeviceError, NativeUnavailable, TunerError

LIB_PATH = Path(__file__).resolve().parent / "_native" / "libhimeno_b200.so"
ABI_VERSION = 2

# enums mirrored from include/himeno_b200.h ---------------------------------
HP_OK, HP_FAIL_PATTERN, HP_FAIL_LAUNCH, HP_TIMEOUT, HP_FAIL_PRESENT = 0, 1, 2, 3, 4
HP_ERR_DEVICE, HP_ERR_ARG, HP_ERR_OOM = -1, -2, -3
NLOOPS, NFIELDS = 13, 14
FIELDS = ("p", "bnd", "wrk1", "wrk2", "a0", "a1", "a2", "a3",
          "b0", "b1", "b2", "c0", "c1", "c2")
FIELD_ID = {name: i for i, name in enumerate(FIELDS)}
VARS = ("p", "bnd", "wrk1", "wrk2", "a", "b", "c", "imax", "jmax", "kmax", "omega",
        "jacobi:nn", "jacobi:gosa", "jacobi:s0", "jacobi:ss", "main:gosa")
VAR_ID = {key: i for i, key in enumerate(VARS)}
K_HOST, K_KERNELS, K_PARALLEL_LOOP, K_PLV, K_COVERED = 0, 1, 2, 3, 4
EV_UPDATE_DEVICE, EV_UPDATE_SELF, EV_DATA_ENTER, EV_DATA_EXIT, EV_DECLARE, EV_PRESENT = 1, 2, 3, 4, 5, 6
BEFORE, AFTER = 0, 1
FLAG_COHERENCE_GUARD = 1
FLAG_FRESH_PROCESS = 2
FLAG_POISON_DEVICE = 4
FLAG_KERNEL_TIMING = 8
FLAG_GRAPH_TIME_LOOP = 16
FLAG_FUSED_TIME_LOOP = 32
FLAG_LITERAL_GOSA = 64
FLAG_HOST_REFERENCE = 128
MAX_SAMPLES = 8
SLAB_HALO = 2      # halo planes per side of a slab context (csrc/decomp.cpp kHalo)


class Grid(C.Structure):
    _fields_ = [("I", C.c_int32), ("J", C.c_int32), ("K", C.c_int32)]


class Event(C.Structure):
    _fields_ = [("loop_id", C.c_int32), ("when", C.c_int32), ("op", C.c_int32),
                ("var", C.c_int32), ("arg", C.c_int32), ("entry", C.c_int32)]


class Schedule(C.Structure):
    _fields_ = [("n_loops", C.c_int32), ("loop_kind", C.c_int32 * NLOOPS),
                ("n_events", C.c_int32), ("events", C.POINTER(Event)),
                ("nn", C.c_int32), ("flags", C.c_int32), ("timeout_s", C.c_double)]


class Result(C.Structure):
    _fields_ = [("wall_s", C.c_double), ("kernel_s", C.c_double), ("host_s", C.c_double),
                ("xfer_s", C.c_double),
                ("h2d_bytes", C.c_uint64), ("d2h_bytes", C.c_uint64),
                ("n_h2d", C.c_uint64), ("n_d2h", C.c_uint64),
                ("n_skipped_stale", C.c_uint64), ("n_implicit", C.c_uint64),
                ("n_launch", C.c_uint64), ("n_stale_reads", C.c_uint64),
                ("gosa", C.c_double), ("samples", C.c_float * MAX_SAMPLES),
                ("n_samples", C.c_int32), ("gosa_f32", C.c_float),
                ("gosa_f32_literal", C.c_int32), ("status", C.c_int32),
                ("diag", C.c_char * 256)]

    def stats(self) -> dict:  # noqa: D401 - plain accessor
        return {"wall_s": self.wall_s, "host_s": self.host_s, "xfer_s": self.xfer_s,
                "h2d_bytes": self.h2d_bytes, "d2h_bytes": self.d2h_bytes,
                "n_h2d": self.n_h2d, "n_d2h": self.n_d2h,
                "n_skipped_stale": self.n_skipped_stale, "n_implicit": self.n_implicit,
                "n_launch": self.n_launch, "n_stale_reads": self.n_stale_reads,
                "gosa": self.gosa, "gosa_f32": self.gosa_f32,
                "gosa_f32_literal": bool(self.gosa_f32_literal),
                "samples": list(self.samples[:self.n_samples]),
                "status": self.status, "diag": self.diag.decode(errors="replace")}


class KernelTimes(C.Structure):
    _fields_ = [("total_ms", C.c_double), ("stencil_ms", C.c_double), ("other_ms", C.c_double),
                ("stencil_iters", C.c_double), ("n_stencil", C.c_int32), ("n_other", C.c_int32)]


# exported symbols: name -> (restype, argtypes); tests check every one exists
_CtxP = C.c_void_p
SIGNATURES = {
    "hp_abi_version": (C.c_int, []),
    "hp_device_count": (C.c_int, []),
    "hp_last_error": (C.c_char_p, []),
    "hp_create": (C.c_int, [C.c_int, C.POINTER(Grid), C.c_int, C.POINTER(_CtxP)]),
    "hp_destroy": (None, [_CtxP]),
    "hp_stream": (C.c_void_p, [_CtxP]),
    "hp_set_samples": (C.c_int, [_CtxP, C.c_int, C.POINTER(C.c_int32)]),
    "hp_run": (C.c_int, [_CtxP, C.POINTER(Schedule), C.POINTER(Result)]),
    "hp_read_field": (C.c_int, [_CtxP, C.c_int, C.c_int, C.c_void_p, C.c_size_t]),
    "hp_write_field": (C.c_int, [_CtxP, C.c_int, C.c_int, C.c_void_p, C.c_size_t]),
    "hp_read_gosa": (C.c_int, [_CtxP, C.c_int, C.POINTER(C.c_double)]),
    "hp_jacobi_device": (C.c_int, [_CtxP, C.c_int, C.c_int]),
    "hp_jacobi_host": (C.c_int, [_CtxP, C.POINTER(C.c_void_p), C.c_int, C.c_int,
                                 C.c_void_p, C.POINTER(C.c_double)]),
    "hp_jacobi_host_async": (C.c_int, [_CtxP, C.POINTER(C.c_void_p), C.c_int, C.c_int,
                                 C.c_void_p, C.POINTER(C.c_double)]),
    "hp_sync": (C.c_int, [_CtxP]),
    "hp_init_device": (C.c_int, [_CtxP]),
    "hp_time_steps": (C.c_int, [_CtxP, C.c_int, C.c_int, C.c_int, C.POINTER(C.c_double)]),
    "hp_time_jacobi": (C.c_int, [_CtxP, C.c_int, C.c_int, C.POINTER(KernelTimes)]),
    "hp_launch_count": (C.c_uint64, [_CtxP]),
    "hp_set_stencil_config": (C.c_int, [C.c_int]),
    "hp_set_temporal_blocking": (C.c_int, [C.c_int]),
    "hp_slab_range": (C.c_int, [C.c_int, C.c_int, C.c_int, C.POINTER(C.c_int32),
                                C.POINTER(C.c_int32)]),
    "hp_create_slab": (C.c_int, [C.c_int, C.POINTER(Grid), C.c_int, C.c_int, C.POINTER(_CtxP)]),
    "hp_group_jacobi": (C.c_int, [C.POINTER(_CtxP), C.c_int, C.c_int, C.POINTER(C.c_double)]),
    "hp_nccl_unique_id": (C.c_int, [C.c_void_p, C.c_size_t]),
    "hp_dd_init": (C.c_int, [_CtxP, C.c_int, C.c_int, C.c_void_p, C.c_size_t]),
    "hp_dd_jacobi": (C.c_int, [_CtxP, C.c_int]),
    "hp_dd_time_steps": (C.c_int, [_CtxP, C.c_int, C.c_int, C.POINTER(C.c_double)]),
    "hp_smem_optin": (C.c_int, [C.c_int, C.c_int, C.POINTER(C.c_int)]),
    "hp_last_two_step_kernel": (C.c_int, []),
    "hp_tx_status": (C.c_int, [_CtxP]),
    "hp_host_alloc": (C.c_void_p, [C.c_size_t]),
    "hp_host_free": (None, [C.c_void_p]),
}

_lib = None
_lock = threading.Lock()


def load(path=None):
    """Load (once) and type the library; raises NativeUnavailable."""
    global _lib
    with _lock:
        if _lib is not None and path is None:
            return _lib
        p = Path(path or os.environ.get("HIMENO_B200_LIB", LIB_PATH))
        if not p.exists():
            raise NativeUnavailable(
                f"{p} not built; run `python -m paper_2002_12115_b200.build` "
                "(there is no CPU fallback for the B200 evaluator)")
        try:
            lib = C.CDLL(str(p))
        except OSError as exc:
            raise NativeUnavailable(f"cannot load {p}: {exc}") from exc
        for name, (res, args) in SIGNATURES.items():
            fn = getattr(lib, name, None)
            if fn is None:
                raise NativeUnavailable(f"{p} lacks symbol {name}")
            fn.restype = res
            fn.argtypes = args
        if lib.hp_abi_version() != ABI_VERSION:
            raise NativeUnavailable(f"{p}: ABI {lib.hp_abi_version()} != {ABI_VERSION}")
        if path is None:
            _lib = lib
        return lib


def nccl_unique_id() -> bytes:
    buf = C.create_string_buffer(128)
    check(load().hp_nccl_unique_id(buf, 128), "hp_nccl_unique_id")
    return buf.raw


def group_jacobi(contexts, nn: int) -> float:
    """Drive slab contexts in-process for nn iterations; returns the global gosa."""
    arr = (C.c_void_p * len(contexts))(*[c.ptr.value for c in contexts])
    g = C.c_double()
    check(load().hp_group_jacobi(arr, len(contexts), nn, C.byref(g)), "hp_group_jacobi")
    return g.value


def smem_optin(kernel_id: int, device: int) -> int:
    """Dynamic shared-memory limit (bytes) of a large-smem kernel on a device."""
    out = C.c_int()
    check(load().hp_smem_optin(kernel_id, device, C.byref(out)), "hp_smem_optin")
    return out.value


def last_two_step_kernel() -> str:
    """Which kernel the most recent two-step pass launched (process-wide)."""
    return {0: "none", 1: "k_stencil_tb2", 2: "k_stencil_tx",
            3: "k_stencil_tb2 (flow)"}[int(load().hp_last_two_step_kernel())]


def last_error() -> str:
    msg = load().hp_last_error()
    return msg.decode(errors="replace") if msg else ""


def device_count() -> int:
    return int(load().hp_device_count())


def check(rc: int, what: str) -> int:
    if rc < 0:
        msg = f"{what}: {last_error()} (rc={rc})"
        if rc == HP_ERR_ARG:
            raise TunerError(msg)
        raise DeviceError(msg)
    return rc


def slab_range(I: int, nranks: int, rank: int) -> tuple:
    """Interior planes [i_begin, i_end) of `rank` (C: hp_slab_range)."""
    b, e = C.c_int32(), C.c_int32()
    check(load().hp_slab_range(I, nranks, rank, C.byref(b), C.byref(e)), "hp_slab_range")
    return b.value, e.value


class Context:
    """One device context (one evaluator worker / one GPU), or one slab of a grid."""

    def __init__(self, device: int, I: int, J: int, K: int, slab=None):
        self.lib = load()
        self.device = device
        ptr = C.c_void_p()
        if slab is None:
            self.shape = (I, J, K)
            self.i_off = 0
            check(self.lib.hp_create(device, C.byref(Grid(I, J, K)), 0, C.byref(ptr)),
                  f"hp_create(device={device}, {I}x{J}x{K})")
        else:
            i_begin, i_end = slab
            self.shape = (i_end - i_begin + 2 * SLAB_HALO, J, K)
            self.i_off = i_begin - SLAB_HALO
            check(self.lib.hp_create_slab(device, C.byref(Grid(I, J, K)), i_begin, i_end,
                                          C.byref(ptr)),
                  f"hp_create_slab(device={device}, planes [{i_begin},{i_end}) of {I})")
        self.global_shape = (I, J, K)
        self._ptr = ptr

    @property
    def ptr(self):
        if self._ptr is None:
            raise TunerError("context destroyed")
        return self._ptr

    def close(self) -> None:
        if getattr(self, "_ptr", None) is not None:
            self.lib.hp_destroy(self._ptr)
            self._ptr = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def __enter__(self):
        return self

    def __exit__(self, *exc):
        self.close()

    @property
    def stream(self) -> int:
        return int(self.lib.hp_stream(self.ptr) or 0)

    def set_samples(self, points) -> None:
        flat = [int(x) for pt in points for x in pt]
        arr = (C.c_int32 * max(1, len(flat)))(*flat)
        check(self.lib.hp_set_samples(self.ptr, len(points), arr), "hp_set_samples")

    def run(self, schedule: Schedule) -> Result:
        res = Result()
        rc = self.lib.hp_run(self.ptr, C.byref(schedule), C.byref(res))
        if rc < 0:
            check(rc, "hp_run")
        return res

    def read_field(self, name: str, side: int = 0):
        import numpy as np
        I, J, K = self.shape
        out = np.empty((I, J, K), dtype=np.float32)
        check(self.lib.hp_read_field(self.ptr, FIELD_ID[name], side,
                                     out.ctypes.data_as(C.c_void_p), out.size), "hp_read_field")
        return out

    def write_field(self, name: str, side: int, values) -> None:
        import numpy as np
        arr = np.ascontiguousarray(values, dtype=np.float32)
        if arr.shape != self.shape:
            raise TunerError(f"field shape {arr.shape} != {self.shape}")
        check(self.lib.hp_write_field(self.ptr, FIELD_ID[name], side,
                                      arr.ctypes.data_as(C.c_void_p), arr.size), "hp_write_field")

    def read_gosa(self, side: int = 1) -> float:
        out = C.c_double()
        check(self.lib.hp_read_gosa(self.ptr, side, C.byref(out)), "hp_read_gosa")
        return out.value

    def tx_status(self) -> int:
        """1 if an exchange-kernel launch of this context timed out (never expected)."""
        return check(self.lib.hp_tx_status(self.ptr), "hp_tx_status")

    def init_device(self) -> None:
        check(self.lib.hp_init_device(self.ptr), "hp_init_device")

    def jacobi_device(self, nn: int, variant: int = 0) -> None:
        check(self.lib.hp_jacobi_device(self.ptr, nn, variant), "hp_jacobi_device")

    def time_steps(self, steps: int, nn: int, variant: int) -> float:
        ms = C.c_double()
        check(self.lib.hp_time_steps(self.ptr, steps, nn, variant, C.byref(ms)), "hp_time_steps")
        return ms.value

    def time_jacobi(self, nn: int, variant: int) -> KernelTimes:
        out = KernelTimes()
        check(self.lib.hp_time_jacobi(self.ptr, nn, variant, C.byref(out)), "hp_time_jacobi")
        return out

    @property
    def launch_count(self) -> int:
        return int(self.lib.hp_launch_count(self.ptr))

    def dd_init(self, nranks: int, rank: int, uid: bytes = b"") -> None:
        buf = C.create_string_buffer(bytes(uid), max(128, len(uid)))
        check(self.lib.hp_dd_init(self.ptr, nranks, rank, buf, len(uid)), "hp_dd_init")

    def dd_jacobi(self, nn: int) -> None:
        check(self.lib.hp_dd_jacobi(self.ptr, nn), "hp_dd_jacobi")

    def dd_time_steps(self, steps: int, nn: int) -> float:
        ms = C.c_double()
        check(self.lib.hp_dd_time_steps(self.ptr, steps, nn, C.byref(ms)), "hp_dd_time_steps")
        return ms.value

    def jacobi_host(self, fields: dict, nn: int, variant: int, p_out) -> float:
        """fields: name -> contiguous float32 [I,J,K] host arrays (numpy); p_out likewise."""
        ptrs = (C.c_void_p * NFIELDS)()
        keep = []
        for name, idx in FIELD_ID.items():
            if name == "wrk2":
                continue
            arr = fields[name]
            keep.append(arr)
            ptrs[idx] = arr.ctypes.data
        g = C.c_double()
        check(self.lib.hp_jacobi_host(self.ptr, ptrs, nn, variant,
                                      C.c_void_p(p_out.ctypes.data), C.byref(g)), "hp_jacobi_host")
        return g.value

    def jacobi_host_async(self, fields: dict, nn: int, variant: int, p_out) -> None:
        """Enqueue jacobi_host without waiting; p_out (pinned for overlap) and gosa are
        delivered by sync()."""
        ptrs = (C.c_void_p * NFIELDS)()
        for name, idx in FIELD_ID.items():
            if name != "wrk2":
                ptrs[idx] = fields[name].ctypes.data
        g = C.c_double()
        check(self.lib.hp_jacobi_host_async(self.ptr, ptrs, nn, variant,
                                            C.c_void_p(p_out.ctypes.data), C.byref(g)),
              "hp_jacobi_host_async")
        # accepted: keep gosa's target and the host buffers alive until sync()
        self._pending_gosa = g
        self._pending_keep = (fields, p_out)

    def sync(self):
        """Wait for the context's queued work; returns the gosa of a pending
        jacobi_host_async call (None if there was none)."""
        check(self.lib.hp_sync(self.ptr), "hp_sync")
        g = getattr(self, "_pending_gosa", None)
        self._pending_gosa = None
        self._pending_keep = None
        return None if g is None else g.value
