"""ctypes binding of libpcr.so (include/pcr.h) — argument marshalling only.

Every step of the hot path runs inside libpcr.so (C++ host control + sm_100a kernels).  This
module only converts Python values to the C-ABI's plain pointers and sizes.  Device buffers
are anything with `.data_ptr()` (torch tensors) or raw integer addresses; streams are
anything with `.cuda_stream` or raw handles.  There is no fallback: if the shared library
is missing the import fails loudly.
"""
from __future__ import annotations

import ctypes
import os

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "libpcr.so")

STATUS = {0: "OK", -1: "INVAL", -2: "NOMEM", -3: "CUDA", -4: "STATE", -5: "NOREQ", -6: "INTERNAL",
          -7: "UNSUPPORTED"}
SHARD_HEADS, SHARD_CONTEXT = 0, 1   # pcr_config.shard_mode (SURVEY §8(e) and its context-split variant)
MODE_OVERLAP, MODE_SYNC, MODE_ONLY_UP, MODE_ONLY_DOWN = 0, 1, 2, 3   # P:703 Up-Down, base, Only-Up, Only-Down
LOAD_SM_GATHER, LOAD_CE_RUNS, LOAD_CE_BLOCKS, LOAD_TMA, LOAD_HYBRID = 0, 1, 2, 3, 4


class PcrError(RuntimeError):
    def __init__(self, status: int, msg: str):
        self.status = status
        self.code = STATUS.get(status, str(status))
        super().__init__(f"pcr {self.code}: {msg}")


class PcrConfig(ctypes.Structure):
    _fields_ = [("n_layers", ctypes.c_int32), ("n_q_heads", ctypes.c_int32), ("n_kv_heads", ctypes.c_int32),
                ("head_dim", ctypes.c_int32), ("rank", ctypes.c_int32), ("world", ctypes.c_int32),
                ("chunk_tokens", ctypes.c_int32), ("page_tokens", ctypes.c_int32),
                ("store_chunks", ctypes.c_int64), ("window", ctypes.c_int32), ("device", ctypes.c_int32),
                ("pool", ctypes.c_void_p), ("pool_bytes", ctypes.c_int64), ("max_inflight", ctypes.c_int32),
                ("max_tokens", ctypes.c_int32), ("gather_ctas", ctypes.c_int32), ("load_mode", ctypes.c_int32),
                ("load_ce_fraction", ctypes.c_float), ("ssd_path", ctypes.c_char_p), ("ssd_chunks", ctypes.c_int64),
                ("shard_mode", ctypes.c_int32)]


class PcrPlan(ctypes.Structure):
    _fields_ = [("n_matched", ctypes.c_int32), ("n_reserved", ctypes.c_int32), ("n1_tokens", ctypes.c_int64),
                ("n2_tokens", ctypes.c_int64), ("slots", ctypes.POINTER(ctypes.c_int32)),
                ("cap_slots", ctypes.c_int32), ("pages", ctypes.POINTER(ctypes.c_int32)),
                ("cap_pages", ctypes.c_int32), ("n_pages", ctypes.c_int32), ("n_evicted", ctypes.c_int32),
                ("evicted_keys", ctypes.POINTER(ctypes.c_uint8)), ("evicted_slots", ctypes.POINTER(ctypes.c_int32)),
                ("cap_evicted", ctypes.c_int32), ("n_from_ssd", ctypes.c_int32)]


class PcrStats(ctypes.Structure):
    _fields_ = [("prefetch_loads", ctypes.c_int64), ("ondemand_loads", ctypes.c_int64),
                ("writebacks", ctypes.c_int64), ("ssd_evictions", ctypes.c_int64),
                ("dram_evictions", ctypes.c_int64), ("ssd_bytes_read", ctypes.c_int64),
                ("ssd_bytes_written", ctypes.c_int64), ("ce_copies", ctypes.c_int64),
                ("ce_layer_loads", ctypes.c_int64), ("sm_layer_loads", ctypes.c_int64)]


class PcrRunOpts(ctypes.Structure):
    _fields_ = [("compute_stream", ctypes.c_void_p), ("load_stream", ctypes.c_void_p),
                ("offload_stream", ctypes.c_void_p), ("comm_stream", ctypes.c_void_p),
                ("gathered_all", ctypes.c_void_p), ("layer_times_ms", ctypes.POINTER(ctypes.c_float)),
                ("mode", ctypes.c_int32), ("host_io", ctypes.c_int32), ("io_ring_layers", ctypes.c_int32),
                ("partial_all", ctypes.POINTER(ctypes.c_float)), ("prefill_done_event", ctypes.c_void_p)]


# Every exported symbol of include/pcr.h with its prototype (restype, argtypes).
_P, _I32, _I64, _VP = ctypes.POINTER, ctypes.c_int32, ctypes.c_int64, ctypes.c_void_p
PROTOTYPES = {
    "pcr_abi_version": (_I32, []),
    "pcr_create": (_I32, [_P(PcrConfig), _P(_VP)]),
    "pcr_destroy": (None, [_VP]),
    "pcr_last_error": (ctypes.c_char_p, [_VP]),
    "pcr_pool_pages": (_I64, [_VP]),
    "pcr_slot_bytes": (_I64, [_VP]),
    "pcr_submit": (_I32, [_VP, _I64, _P(ctypes.c_uint32), _I64, _I64]),
    "pcr_match_prefix": (_I32, [_VP, _I64, _P(_I64), _I32, _P(PcrPlan)]),
    "pcr_release": (_I32, [_VP, _I64, _I32]),
    "pcr_store_write": (_I32, [_VP, _I32, _VP]),
    "pcr_store_read": (_I32, [_VP, _I32, _VP]),
    "pcr_leaf_list": (_I32, [_VP, _P(ctypes.c_uint8), _I32, _P(_I32)]),
    "pcr_blake2b": (_I32, [_VP, _I64, _VP, _I32, _I32, _P(ctypes.c_uint8)]),
    "pcr_load_layer_kv": (_I32, [_VP, _I64, _I32, _VP]),
    "pcr_prefill_attn_layer": (_I32, [_VP, _I64, _I32, _VP, _VP, _VP, _VP, _VP]),
    "pcr_run_prefill": (_I32, [_VP, _I64, _VP, _VP, _VP, _VP, _VP, _VP, _I32, _P(ctypes.c_float)]),
    "pcr_kernel_launches": (_I64, [_VP]),
    "pcr_set_load_mode": (_I32, [_VP, _I32, ctypes.c_float]),
    "pcr_merge_partials": (_I32, [_VP, _VP, _I32, _I64, _VP, _VP]),
    "pcr_comm_unique_id": (_I32, [_P(ctypes.c_uint8)]),
    "pcr_comm_init": (_I32, [_VP, _P(ctypes.c_uint8)]),
    "pcr_run_prefill_sharded": (_I32, [_VP, _I64, _VP, _VP, _VP, _VP, _VP, _VP, _VP, _VP, _I32,
                                       _P(ctypes.c_float)]),
    "pcr_offload_layer_kv": (_I32, [_VP, _I64, _I32, _VP]),
    "pcr_run_prefill_ex": (_I32, [_VP, _I64, _VP, _VP, _VP, _VP, _P(PcrRunOpts)]),
    "pcr_get_stats": (_I32, [_VP, _P(PcrStats)]),
}

_lib = None


def load_library(path: str = None):
    """Load libpcr.so (PCR_LIB_PATH overrides the in-tree build, e.g. the sanitizer build the
    tests make).  Fails loudly when it is missing: there is no fallback."""
    global _lib
    if path is None:
        path = os.environ.get("PCR_LIB_PATH", LIB_PATH)
    if _lib is None:
        if not os.path.exists(path):
            raise ImportError(f"{path} not built: run `python -m paper_2603_23049_b200.build` "
                              "(the CUDA path has no fallback)")
        lib = ctypes.CDLL(path)
        for name, (res, args) in PROTOTYPES.items():
            f = getattr(lib, name)
            f.restype, f.argtypes = res, args
        _lib = lib
    return _lib


def _ptr(x):
    if x is None:
        return None
    if hasattr(x, "data_ptr"):
        return ctypes.c_void_p(x.data_ptr())
    return ctypes.c_void_p(int(x))


def _stream(s):
    if s is None:
        return None
    if hasattr(s, "cuda_stream"):
        return ctypes.c_void_p(s.cuda_stream)
    return ctypes.c_void_p(int(s))


def _event(e):
    """cudaEvent_t handle of a torch.cuda.Event (or a raw handle), None passes through."""
    if e is None:
        return None
    if hasattr(e, "cuda_event"):
        return ctypes.c_void_p(e.cuda_event)
    return ctypes.c_void_p(int(e))


def blake2b(data: bytes, digest_len: int = 64, key: bytes = b"") -> bytes:
    lib = load_library()
    out = (ctypes.c_uint8 * digest_len)()
    st = lib.pcr_blake2b(data, len(data), key if key else None, len(key), digest_len, out)
    if st != 0:
        raise PcrError(st, "pcr_blake2b")
    return bytes(out)


def comm_unique_id() -> bytes:
    """ncclGetUniqueId through libpcr (create on one rank, broadcast the 128 bytes)."""
    lib = load_library()
    out = (ctypes.c_uint8 * 128)()
    st = lib.pcr_comm_unique_id(out)
    if st != 0:
        raise PcrError(st, "pcr_comm_unique_id")
    return bytes(out)


class Context:
    """One pcr_ctx.  `device=-1` gives a host-control-only context (no CUDA calls)."""

    def __init__(self, n_layers, n_q_heads, n_kv_heads, head_dim, chunk_tokens, page_tokens, store_chunks,
                 window, device=-1, pool=None, pool_bytes=None, rank=0, world=1, max_inflight=0, max_tokens=0,
                 gather_ctas=0, load_mode=LOAD_SM_GATHER, ssd_path=None, ssd_chunks=0, load_ce_fraction=0.0,
                 shard_mode=SHARD_HEADS):
        self.lib = load_library()
        if pool_bytes is None:
            pool_bytes = pool.numel() * pool.element_size() if hasattr(pool, "numel") else 0
        self._pool = pool
        self._ssd_path = ssd_path.encode() if isinstance(ssd_path, str) else ssd_path
        cfg = PcrConfig(n_layers, n_q_heads, n_kv_heads, head_dim, rank, world, chunk_tokens, page_tokens,
                        store_chunks, window, device, _ptr(pool), int(pool_bytes), max_inflight, max_tokens,
                        gather_ctas, load_mode, float(load_ce_fraction), self._ssd_path, ssd_chunks, shard_mode)
        h = ctypes.c_void_p()
        st = self.lib.pcr_create(ctypes.byref(cfg), ctypes.byref(h))
        if st != 0:
            raise PcrError(st, "pcr_create")
        self.h = h
        self.cfg = cfg
        self.C, self.S = chunk_tokens, page_tokens
        self.n_layers = n_layers

    def close(self):
        if getattr(self, "h", None):
            self.lib.pcr_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def _check(self, st, what):
        if st != 0:
            raise PcrError(st, f"{what}: {self.lib.pcr_last_error(self.h).decode()}")

    @property
    def pool_pages(self):
        return int(self.lib.pcr_pool_pages(self.h))

    @property
    def slot_bytes(self):
        return int(self.lib.pcr_slot_bytes(self.h))

    @property
    def stats(self):
        st = PcrStats()
        self._check(self.lib.pcr_get_stats(self.h, ctypes.byref(st)), "pcr_get_stats")
        return {f: getattr(st, f) for f, _ in PcrStats._fields_}

    def set_load_mode(self, load_mode, load_ce_fraction=0.0):
        self._check(self.lib.pcr_set_load_mode(self.h, int(load_mode), float(load_ce_fraction)), "pcr_set_load_mode")

    @property
    def kernel_launches(self):
        return int(self.lib.pcr_kernel_launches(self.h))

    def submit(self, req_id, tokens, n_cacheable=None):
        t = np.ascontiguousarray(tokens, dtype=np.uint32)
        n_cacheable = len(t) if n_cacheable is None else n_cacheable
        self._check(self.lib.pcr_submit(self.h, req_id, t.ctypes.data_as(_P(ctypes.c_uint32)), len(t), n_cacheable),
                    "pcr_submit")

    def match_prefix(self, req_id, pending=(), cap_chunks=4096, cap_pages=1 << 16):
        pend = np.ascontiguousarray(list(pending), dtype=np.int64)
        slots = np.zeros(cap_chunks, np.int32)
        pages = np.zeros(cap_pages, np.int32)
        ev_keys = np.zeros((cap_chunks, 16), np.uint8)
        ev_slots = np.zeros(cap_chunks, np.int32)
        plan = PcrPlan()
        plan.slots = slots.ctypes.data_as(_P(ctypes.c_int32))
        plan.cap_slots = cap_chunks
        plan.pages = pages.ctypes.data_as(_P(ctypes.c_int32))
        plan.cap_pages = cap_pages
        plan.evicted_keys = ev_keys.ctypes.data_as(_P(ctypes.c_uint8))
        plan.evicted_slots = ev_slots.ctypes.data_as(_P(ctypes.c_int32))
        plan.cap_evicted = cap_chunks
        self._check(self.lib.pcr_match_prefix(self.h, req_id, pend.ctypes.data_as(_P(_I64)) if len(pend) else None,
                                              len(pend), ctypes.byref(plan)), "pcr_match_prefix")
        nm, nr, ne = plan.n_matched, plan.n_reserved, plan.n_evicted
        return dict(n_matched=nm, n_reserved=nr, n1=plan.n1_tokens, n2=plan.n2_tokens, n_from_ssd=plan.n_from_ssd,
                    slots=slots[:nm + nr].tolist(), pages=pages[:plan.n_pages].tolist(),
                    evicted=[(bytes(ev_keys[i]), int(ev_slots[i])) for i in range(ne)])

    def release(self, req_id, commit=True):
        self._check(self.lib.pcr_release(self.h, req_id, 1 if commit else 0), "pcr_release")

    def store_write(self, slot, data):
        a = np.ascontiguousarray(data)
        if a.nbytes != self.slot_bytes:
            raise ValueError(f"slot record must be {self.slot_bytes} bytes, got {a.nbytes}")
        self._check(self.lib.pcr_store_write(self.h, slot, a.ctypes.data), "pcr_store_write")

    def store_read(self, slot):
        a = np.empty(self.slot_bytes // 2, np.uint16)
        self._check(self.lib.pcr_store_read(self.h, slot, a.ctypes.data), "pcr_store_read")
        return a

    def leaf_list(self):
        n = ctypes.c_int32()
        cap = 1 << 16
        buf = np.zeros((cap, 16), np.uint8)
        self._check(self.lib.pcr_leaf_list(self.h, buf.ctypes.data_as(_P(ctypes.c_uint8)), cap, ctypes.byref(n)),
                    "pcr_leaf_list")
        return [bytes(buf[i]) for i in range(n.value)]

    # ---- device path ---------------------------------------------------------------
    def load_layer_kv(self, req_id, layer, load_stream):
        self._check(self.lib.pcr_load_layer_kv(self.h, req_id, layer, _stream(load_stream)), "pcr_load_layer_kv")

    def prefill_attn_layer(self, req_id, layer, q, k_new, v_new, out, compute_stream):
        self._check(self.lib.pcr_prefill_attn_layer(self.h, req_id, layer, _ptr(q), _ptr(k_new), _ptr(v_new),
                                                    _ptr(out), _stream(compute_stream)), "pcr_prefill_attn_layer")

    def run_prefill(self, req_id, q_all, k_all, v_all, out_all, compute_stream, load_stream=None,
                    mode=MODE_OVERLAP, layer_times=False):
        times = (ctypes.c_float * (2 * self.n_layers))() if layer_times else None
        self._check(self.lib.pcr_run_prefill(self.h, req_id, _ptr(q_all), _ptr(k_all), _ptr(v_all), _ptr(out_all),
                                             _stream(compute_stream), _stream(load_stream), mode, times),
                    "pcr_run_prefill")
        if layer_times:
            t = np.array(times[:], dtype=np.float64).reshape(self.n_layers, 2)
            return t
        return None

    def offload_layer_kv(self, req_id, layer, offload_stream):
        self._check(self.lib.pcr_offload_layer_kv(self.h, req_id, layer, _stream(offload_stream)),
                    "pcr_offload_layer_kv")

    def run_prefill_ex(self, req_id, q_all, k_all, v_all, out_all, compute_stream, load_stream=None,
                       offload_stream=None, comm_stream=None, gathered_all=None, mode=MODE_OVERLAP,
                       layer_times=False, host_io=False, io_ring_layers=0, partial_all=None,
                       prefill_done_event=None):
        """Full pipeline (P:480 three streams): returns [L][3] ms (gather, append+attn, offload) if
        layer_times, else None.  host_io: q/k/v/out are page-locked HOST tensors; the library
        stages them per layer on its own copy streams (the e2e path)."""
        times = (ctypes.c_float * (3 * self.n_layers))() if layer_times else None
        o = PcrRunOpts(_stream(compute_stream), _stream(load_stream), _stream(offload_stream),
                       _stream(comm_stream), _ptr(gathered_all),
                       ctypes.cast(times, _P(ctypes.c_float)) if times is not None else None, mode,
                       1 if host_io else 0, int(io_ring_layers),
                       ctypes.cast(_ptr(partial_all), _P(ctypes.c_float)) if partial_all is not None else None,
                       _event(prefill_done_event))
        self._check(self.lib.pcr_run_prefill_ex(self.h, req_id, _ptr(q_all), _ptr(k_all), _ptr(v_all),
                                                _ptr(out_all), ctypes.byref(o)), "pcr_run_prefill_ex")
        if layer_times:
            return np.array(times[:], dtype=np.float64).reshape(self.n_layers, 3)
        return None

    def merge_partials(self, gathered, n_parts, n2, out, stream):
        """shard_mode 1: merge n_parts partial blocks (fp32 device tensor) into bf16 `out`."""
        self._check(self.lib.pcr_merge_partials(self.h, _ptr(gathered), int(n_parts), int(n2), _ptr(out),
                                                _stream(stream)), "pcr_merge_partials")

    def comm_init(self, uid: bytes):
        buf = (ctypes.c_uint8 * 128).from_buffer_copy(uid)
        self._check(self.lib.pcr_comm_init(self.h, buf), "pcr_comm_init")

    def run_prefill_sharded(self, req_id, q_all, k_all, v_all, out_all, gathered_all, compute_stream,
                            load_stream, comm_stream, mode=MODE_OVERLAP, layer_times=False):
        times = (ctypes.c_float * (2 * self.n_layers))() if layer_times else None
        self._check(self.lib.pcr_run_prefill_sharded(self.h, req_id, _ptr(q_all), _ptr(k_all), _ptr(v_all),
                                                     _ptr(out_all), _ptr(gathered_all), _stream(compute_stream),
                                                     _stream(load_stream), _stream(comm_stream), mode, times),
                    "pcr_run_prefill_sharded")
        if layer_times:
            return np.array(times[:], dtype=np.float64).reshape(self.n_layers, 2)
        return None
