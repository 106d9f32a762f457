"""ctypes binding of libsrflow.so (include/srflow.h).

This is the only module that touches the C ABI.  There is no CPU fallback:
if the shared object is missing or a device call fails, the call raises.
Status codes are translated into the exception classes of :mod:`.errors`
(the same hierarchy as the reference's errors.py).
"""
from __future__ import annotations

import ctypes as C
import os
import threading

from . import errors

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "lib", "libsrflow.so")

SRF_OK = 0
SRF_PENDING = 1
PUT_WAIT_EMPTY = 0x1
APPLY_XOR = 0
APPLY_SGD = 1
MAX_WORKERS = 16

_STATUS = {
    10: errors.ZeroLength,
    11: errors.OutOfMemory,
    12: errors.OutOfBounds,
    13: errors.NotRegistered,
    14: errors.BadToken,
    15: errors.RemoteOutOfBounds,
    16: errors.InvalidLength,
    17: errors.Timeout,
    18: errors.PeerUnreachable,
    19: errors.InvalidConfig,
    20: errors.ShapeMismatch,
    21: errors.ProtocolError,
    22: errors.DeviceError,
}

u64 = C.c_uint64
i64 = C.c_int64
vp = C.c_void_p
P = C.POINTER

# name -> (restype, argtypes); mirrors include/srflow.h one for one
SIGNATURES = {
    "srf_last_error": (C.c_char_p, []),
    "srf_version": (C.c_int, []),
    "srf_device_count": (C.c_int, [P(C.c_int)]),
    "srf_launch_count": (u64, []),
    "srf_host_alloc": (C.c_int, [u64, P(vp)]),
    "srf_host_free": (C.c_int, [vp]),
    "srf_tune": (C.c_int, [C.c_int, C.c_int]),
    "srf_space_create": (C.c_int, [C.c_int, C.c_int, u64, C.c_uint32, P(vp)]),
    "srf_space_destroy": (C.c_int, [vp]),
    "srf_space_info": (C.c_int, [vp, P(C.c_int), P(C.c_int), P(u64), P(vp)]),
    "srf_space_cuda_stream": (vp, [vp]),
    "srf_region_alloc": (C.c_int, [vp, u64, C.c_int, u64, P(i64), P(u64)]),
    "srf_region_count": (C.c_int, [vp, P(C.c_uint32)]),
    "srf_next_addr": (C.c_int, [vp, P(u64)]),
    "srf_check_remote": (C.c_int, [vp, u64, u64, u64]),
    "srf_check_registered": (C.c_int, [vp, u64, u64, u64]),
    "srf_read": (C.c_int, [vp, u64, u64, vp]),
    "srf_write": (C.c_int, [vp, u64, u64, vp]),
    "srf_write_async": (C.c_int, [vp, u64, u64, vp, vp]),
    "srf_read_async": (C.c_int, [vp, u64, u64, vp, vp]),
    "srf_device_ptr": (C.c_int, [vp, u64, P(vp)]),
    "srf_space_sync": (C.c_int, [vp]),
    "srf_connect": (C.c_int, [vp, vp]),
    "srf_space_export": (C.c_int, [vp, vp]),
    "srf_space_export_fd": (C.c_int, [vp, P(C.c_int)]),
    "srf_space_import_fd": (C.c_int, [C.c_int, C.c_int, C.c_int, u64, P(vp)]),
    "srf_enable_peer": (C.c_int, [C.c_int, C.c_int]),
    "srf_space_import": (C.c_int, [vp, C.c_int, C.c_int, u64, P(vp)]),
    "srf_region_import": (C.c_int, [vp, i64, u64, u64, C.c_int, u64]),
    "srf_stream_create": (C.c_int, [vp, P(vp)]),
    "srf_stream_destroy": (C.c_int, [vp]),
    "srf_stream_cuda": (vp, [vp]),
    "srf_stream_sync": (C.c_int, [vp]),
    "srf_event_record": (C.c_int, [vp, vp, P(vp)]),
    "srf_event_query": (C.c_int, [vp]),
    "srf_event_wait": (C.c_int, [vp]),
    "srf_event_free": (C.c_int, [vp]),
    "srf_event_wait_free": (C.c_int, [vp]),
    "srf_graph_begin": (C.c_int, [vp]),
    "srf_graph_end": (C.c_int, [vp, P(vp)]),
    "srf_graph_launch": (C.c_int, [vp, vp]),
    "srf_graph_destroy": (C.c_int, [vp]),
    "srf_stream_wait_event": (C.c_int, [vp, vp]),
    "srf_space_wait_event": (C.c_int, [vp, vp]),
    "srf_timing_event_create": (C.c_int, [vp, P(vp)]),
    "srf_event_record_on": (C.c_int, [vp, vp]),
    "srf_event_elapsed_ms": (C.c_int, [vp, vp, P(C.c_float)]),
    "srf_put": (C.c_int, [vp, P(u64), P(u64), P(u64), C.c_int, vp, u64, u64,
                          C.c_int, vp, P(vp)]),
    "srf_get": (C.c_int, [vp, u64, u64, vp, u64, u64, u64, vp, P(vp)]),
    "srf_put_inline": (C.c_int, [vp, u64, u64, C.c_char_p, C.c_uint32, vp, u64, u64, C.c_int, vp,
                                 P(vp)]),
    "srf_put_consume": (C.c_int, [vp, P(u64), P(u64), P(u64), C.c_int, vp, u64, u64, C.c_int,
                                  vp, u64, vp, P(vp)]),
    "srf_copy": (C.c_int, [vp, u64, u64, u64, vp, P(vp)]),
    "srf_flag_wait": (C.c_int, [vp, u64, C.c_uint8, C.c_int, u64, vp]),
    "srf_apply": (C.c_int, [vp, u64, u64, P(vp), P(u64), C.c_int, C.c_int,
                            C.c_float, vp, P(vp)]),
    "srf_consume_checksum": (C.c_int, [vp, u64, u64, u64, u64, u64, vp]),
    "srf_batch_put_create": (C.c_int, [C.c_int, P(vp), P(u64), P(u64), P(u64), P(u64), P(vp),
                                       P(u64), P(u64), C.c_int, P(vp)]),
    "srf_batch_gen_create": (C.c_int, [C.c_int, P(vp), P(u64), P(u64), P(u64), P(vp), P(u64),
                                       P(u64), u64, P(vp)]),
    "srf_batch_apply_create": (C.c_int, [vp, C.c_int, P(u64), P(u64), P(C.c_int), P(C.c_int),
                                         P(vp), P(u64), P(C.c_int), P(vp), P(u64), P(u64),
                                         P(u64), C.c_int, C.c_float, P(vp)]),
    "srf_batch_launch": (C.c_int, [vp, vp, u64, C.c_int, C.c_int]),
    "srf_batch_destroy": (C.c_int, [vp]),
    "srf_batch_set_iteration_source": (C.c_int, [vp, vp, u64]),
    "srf_counter_add": (C.c_int, [vp, u64, u64, vp]),
    "srf_ps_persistent": (C.c_int, [vp, vp, vp, P(vp), C.c_int, vp, u64, C.c_uint32, C.c_int]),
    "srf_batch_gen_set_meta": (C.c_int, [vp, C.c_int, P(C.c_int), vp]),
    "srf_dyn_recv": (C.c_int, [vp, u64, C.c_int, vp, u64, u64, u64, u64, u64, u64, vp]),
    "srf_torch_pool_attach": (C.c_int, [vp, u64, u64]),
    "srf_torch_pool_stats": (C.c_int, [C.c_int, P(u64), P(u64), P(u64)]),
    "srf_torch_malloc": (vp, [C.c_ssize_t, C.c_int, vp]),
    "srf_torch_free": (None, [vp, C.c_ssize_t, C.c_int, vp]),
    "srf_batch_gen_set_offsets": (C.c_int, [vp, P(u64)]),
    "srf_batch_gen_set_ready": (C.c_int, [vp, P(vp), P(u64)]),
    "srf_batch_apply_set_ready": (C.c_int, [vp, vp, P(u64)]),
    "srf_batch_apply_set_forward": (C.c_int, [vp, P(C.c_int), P(vp), P(u64), P(u64), vp, u64]),
    "srf_batch_put_set_src_ready": (C.c_int, [vp, P(vp), P(u64)]),
    "srf_ps_exchange_create": (C.c_int, [vp, P(u64), vp, P(u64), P(vp), C.c_int, P(u64),
                                         P(vp)]),
    "srf_ps_exchange_launch": (C.c_int, [vp, vp, u64, C.c_int]),
    "srf_ps_exchange_destroy": (C.c_int, [vp]),
    "srf_ps_exchange_link": (C.c_int, [vp, P(C.c_int)]),
    "srf_ps_exchange_launch_n": (C.c_int, [vp, vp, u64, C.c_uint32, C.c_int]),
    "srf_doorbell_bind": (C.c_int, [vp, u64, u64, C.c_int]),
    "srf_flag_read": (C.c_int, [vp, u64, u64, vp]),
    "srf_flag_clear": (C.c_int, [vp, u64]),
    "srf_rpc_transfer": (C.c_int, [vp, u64, C.c_uint32, u64, u64, u64, vp, u64, u64, u64, u64,
                                   u64, vp, vp]),
    "srf_reduce_max_f32": (C.c_int, [vp, u64, u64, u64, vp]),
    "srf_concat_tile": (C.c_int, [vp, C.c_int, P(u64), P(u64), u64, u64, vp]),
    "srf_add_bcast": (C.c_int, [vp, C.c_int, u64, P(u64), u64, P(u64), C.c_int, u64, vp]),
    "srf_gen_reference": (C.c_int, [vp, u64, u64, u64, u64, u64, u64, vp, P(vp)]),
    "srf_edge_create": (C.c_int, [vp, u64, u64, u64, C.c_uint32, u64, vp, u64, u64, C.c_uint32,
                                  u64, u64, P(vp)]),
    "srf_edge_info": (C.c_int, [vp, P(u64), P(C.c_uint32), P(C.c_int), P(u64)]),
    "srf_edge_send": (C.c_int, [vp, C.c_uint32, vp, vp]),
    "srf_edge_state": (C.c_int, [vp, P(C.c_uint32), C.c_uint32]),
    "srf_edge_consume": (C.c_int, [vp, u64, C.c_uint32, u64, u64, u64, C.c_uint32, C.c_int, u64,
                                   vp, u64, vp]),
    "srf_edge_destroy": (C.c_int, [vp]),
    "srf_edge_create_pull": (C.c_int, [vp, u64, u64, u64, C.c_uint32, u64, vp, u64, u64,
                                       C.c_uint32, u64, u64, u64, C.c_int, P(vp)]),
    "srf_edge_recv": (C.c_int, [vp, C.c_uint32, vp, vp]),
    "srf_edge_post": (C.c_int, [vp, vp, u64, u64, u64, C.c_uint32, vp]),
    "srf_dyn_edge_create": (C.c_int, [vp, u64, u64, u64, u64, C.c_uint32, vp, u64, u64,
                                      C.c_uint32, u64, u64, P(vp)]),
    "srf_dyn_edge_recv": (C.c_int, [vp, C.c_uint32, vp, vp]),
    "srf_dyn_edge_consume": (C.c_int, [vp, vp, u64, C.c_uint32, C.c_int, u64, vp]),
    "srf_dyn_edge_send": (C.c_int, [vp, vp, u64, u64, C.c_uint32, C.c_uint32, C.c_int, P(u64),
                                    u64, u64, C.c_uint32, u64, u64, C.c_uint32, vp]),
    "srf_dyn_edge_destroy": (C.c_int, [vp]),
    "srf_matmul": (C.c_int, [C.c_int, u64, u64, u64, u64, u64, u64, vp]),
    "srf_compute": (C.c_int, [vp, C.c_int, C.c_int, u64, u64, u64, u64, u64, u64, vp]),
    "srf_record_begin": (C.c_int, []),
    "srf_record_taint": (C.c_int, [C.c_char_p]),
    "srf_record_end": (C.c_int, [P(vp), P(C.c_int)]),
    "srf_oplist_info": (C.c_int, [vp, P(C.c_uint32), P(C.c_int), C.c_char_p, C.c_uint32]),
    "srf_oplist_same": (C.c_int, [vp, vp, C.c_int64]),
    "srf_oplist_diff": (C.c_int, [vp, vp, C.c_int64, C.c_char_p, C.c_uint32]),
    "srf_oplist_replay": (C.c_int, [vp, u64, C.c_uint32, vp]),
    "srf_oplist_destroy": (C.c_int, [vp]),
    "srf_replay_set_create": (C.c_int, [P(vp), P(C.c_int64), C.c_uint32, P(vp)]),
    "srf_replay_set_launch": (C.c_int, [vp, C.c_uint32, u64, vp]),
    "srf_replay_set_info": (C.c_int, [vp, P(C.c_uint32), P(C.c_uint32), P(C.c_uint32), P(u64)]),
    "srf_replay_set_destroy": (C.c_int, [vp]),
}

_lib = None
_lock = threading.Lock()


def load() -> C.CDLL:
    """Load libsrflow.so (raises if it was not built)."""
    global _lib
    if _lib is not None:
        return _lib
    with _lock:
        if _lib is None:
            if not os.path.exists(LIB_PATH):
                raise ImportError(
                    f"{LIB_PATH} is missing: build it with "
                    f"`python -m paper_1805_08430_b200.build` (no CPU fallback exists)")
            lib = C.CDLL(LIB_PATH)
            for name, (res, args) in SIGNATURES.items():
                fn = getattr(lib, name)
                fn.restype = res
                fn.argtypes = args
            _lib = lib
            _apply_env_knobs(lib)
    return _lib


_KNOBS = {"SRFLOW_CTAS_PER_SM": 0, "SRFLOW_COPY_THREADS": 1, "SRFLOW_PUT_IMPL": 2,
          "SRFLOW_ALLOC_VMM": 3, "SRFLOW_UNROLL": 4, "SRFLOW_VEC32": 5,
          "SRFLOW_PEER_CE_KIB": 6, "SRFLOW_FORCE_SYS": 7, "SRFLOW_PUT_TIMEOUT_MS": 8,
          "SRFLOW_EDGE_CTAS_PER_SM": 9, "SRFLOW_EDGE_CHUNK_KIB": 10,
          "SRFLOW_CONSUME_THREADS": 11, "SRFLOW_GEN_UNIT_KIB": 12,
          "SRFLOW_CONSUME_RELEASE": 13, "SRFLOW_EDGE_CTAS": 14,
          "SRFLOW_PULL_NO_PREFETCH": 16}


def _apply_env_knobs(lib) -> None:
    """Launch-geometry / implementation knobs from the environment."""
    for name, knob in _KNOBS.items():
        if name in os.environ:
            rc = lib.srf_tune(knob, int(os.environ[name]))
            if rc != SRF_OK:
                raise errors.InvalidConfig(f"{name}={os.environ[name]}: "
                                           f"{lib.srf_last_error().decode()}")


def tune(knob: str, value: int) -> None:
    call("srf_tune", {"ctas_per_sm": 0, "copy_threads": 1, "put_impl": 2,
                      "alloc_vmm": 3, "unroll": 4, "vec32": 5,
                      "peer_ce_kib": 6, "force_sys": 7, "put_timeout_ms": 8,
                      "edge_ctas_per_sm": 9, "edge_chunk_kib": 10,
                      "consume_threads": 11, "gen_unit_kib": 12,
                      "consume_release": 13, "edge_ctas": 14,
                      "pull_no_prefetch": 16}[knob], value)


def last_error() -> str:
    msg = load().srf_last_error()
    return msg.decode(errors="replace") if msg else ""


def check(rc: int) -> int:
    """Raise the errors.py class mapped from a non-OK status."""
    if rc == SRF_OK or rc == SRF_PENDING:
        return rc
    cls = _STATUS.get(rc, errors.DeviceError)
    raise cls(last_error())


def call(name: str, *args) -> int:
    return check(getattr(load(), name)(*args))


def u64_array(values) -> "C.Array":
    values = list(values)
    return (u64 * max(1, len(values)))(*values)


def launch_count() -> int:
    return int(load().srf_launch_count())


def device_count() -> int:
    n = C.c_int(0)
    rc = load().srf_device_count(C.byref(n))
    return n.value if rc == SRF_OK else 0


class PinnedBuffer:
    """Page-locked host bytes (cudaHostAlloc) for asynchronous H2D staging."""

    def __init__(self, nbytes: int):
        p = C.c_void_p()
        call("srf_host_alloc", nbytes, C.byref(p))
        self.ptr = p.value
        self.nbytes = nbytes

    def write(self, data: bytes) -> None:
        C.memmove(self.ptr, data, len(data))

    def __del__(self):  # pragma: no cover
        try:
            load().srf_host_free(C.c_void_p(self.ptr))
        except Exception:
            pass


class Event:
    """Completion of one verb (a CUDA event recorded after its kernel)."""

    __slots__ = ("_h",)

    def __init__(self, handle):
        self._h = handle

    def query(self) -> bool:
        if self._h is None:
            return True
        return call("srf_event_query", self._h) == SRF_OK

    def wait(self) -> None:
        if self._h is not None:
            call("srf_event_wait", self._h)

    def free(self) -> None:
        if self._h is not None:
            load().srf_event_free(self._h)
            self._h = None

    def wait_free(self) -> None:
        """wait() then free() in one call (the event returns to the pool)."""
        if self._h is not None:
            h, self._h = self._h, None
            check(load().srf_event_wait_free(h))

    def __del__(self):  # pragma: no cover - interpreter teardown order
        try:
            self.free()
        except Exception:
            pass
